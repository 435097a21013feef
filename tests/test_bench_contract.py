"""bench.py's reference arm and the line contract both arms share (CPU only).

The driver computes the GPU/reference ratio only when both arms print the same `metric`
(BASELINE.json) and `unit`; under torchrun only rank 0 of the reference arm prints."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _run(cmd, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    return p.stdout


def test_reference_arm_line():
    out = _run([sys.executable, "bench.py", "--impl", "reference", "--workload", "llama7b_small",
                "--steps", "1", "--warmup", "3"])
    lines = _lines(out)
    assert len(lines) == 1
    d = lines[0]
    baseline = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    sys.path.insert(0, ROOT)
    import bench
    assert d["impl"] == "reference"
    assert d["metric"] == baseline["metric"] == bench.METRIC
    assert d["unit"] == bench.UNIT and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("reference", "port") and cb["cores"] >= 1
    assert d["cpu_single_thread"]["cores"] == 1


@pytest.mark.timeout(900)
def test_reference_arm_under_torchrun_prints_once():
    out = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--impl",
                "reference", "--gpus", "2", "--workload", "llama7b_small", "--steps", "1",
                "--warmup", "3"])
    lines = _lines(out)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


@pytest.mark.gpu
def test_gpu_arm_line():
    """The GPU arm on a small workload: same metric/unit as the reference arm, parity checked,
    roofline / e2e / launch-count fields present."""
    out = _run_gpu([sys.executable, "bench.py", "--workload", "llama7b_small", "--steps", "3",
                    "--warmup", "3", "--no-cpu-baseline"])
    lines = _lines(out)
    assert len(lines) == 1
    d = lines[0]
    sys.path.insert(0, ROOT)
    import bench
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT and d["n_gpus"] == 1
    assert d["value"] > 0 and d["parity"].startswith("ok")
    assert d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])


def _run_gpu(cmd, timeout=600):
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    return p.stdout
