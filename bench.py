#!/usr/bin/env python3
"""Benchmark of the B200 bipolar-INT WnAm GEMM (arXiv 2409.17870 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload ffn70b|sweep4096|w2a4_4096|llama7b|llama7b_small|decode]

Default workload = BASELINE.json configs[4], the largest single-GPU configuration: the
Llama-2-70B FFN projection W[28672 x 8192] W2A4 against X[4096 tokens x 8192] A4. One
step = that GEMM through the C ABI (apmm_cu_matmul_ap: packed bit planes in HBM -> int32 Y
in HBM). Metric = effective TOPS = 2*M*N*K / device time (BASELINE.json `metric`).

Multi-GPU: `--gpus N` (N > 1) re-launches itself under torch.distributed.run with one
process per GPU unless it already runs under torchrun. ffn70b is N-sharded:
rank p owns the contiguous W row block p of 28672/N rows, X is replicated, the GEMMs are
independent ("scaling": "strong": the whole job is the one full GEMM), `value` is the full
GEMM's ops / max-over-ranks compute time. The optional all-gather of the int32 row blocks
(NCCL over NVLink, only where the consumer needs the full output) is timed separately and
reported under "gather". Every other workload runs the same GEMMs on each rank as
independent replicas ("scaling": "weak").

`--impl reference` times the reference's own CPU matmul_ap (oracle/_ref, compiled from
/root/reference/proj/src) on the same config, row-sliced over all host threads (legal per
SPEC.md:266), plus the as-shipped 1-thread figure; only rank 0 runs it.

After the timed region the GPU arm compares sampled rows of every Y it timed against the
reference's matmul_ap (`"parity"` in the line); a mismatch exits non-zero.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# One metric string, identical in both arms (BASELINE.json `metric`).
METRIC = "effective TOPS (2MNK/s) of WnAm bipolar-INT GEMM vs roofline; decode HBM GB/s"
UNIT = "TOPS"

# ----------------------------------------------------------------------------- workloads
SWEEP_BITS = [(nw, nx) for nw in (1, 2, 3, 4) for nx in (2, 4, 8)]


def workload_gemms(name: str):
    """List of (rows_w=N_out, rows_x=M_tok, K, n_w, n_x) in reference orientation
    matmul_ap(W[N_out x K], X[M_tok x K]) -> Y[N_out x M_tok]."""
    if name == "ffn70b":
        return [(28672, 4096, 8192, 2, 4)]
    if name == "sweep4096":
        return [(4096, 4096, 4096, nw, nx) for nw, nx in SWEEP_BITS]
    if name == "w2a4_4096":
        return [(4096, 4096, 4096, 2, 4)]
    if name == "llama7b":
        return [(n, m, k, 2, 4) for (n, k) in ((4096, 4096), (11008, 4096), (4096, 11008))
                for m in (2048,)]
    if name == "llama7b_small":
        return [(n, m, k, 2, 4) for (n, k) in ((4096, 4096), (11008, 4096), (4096, 11008))
                for m in (1, 16)]
    if name == "llama7b_mid":
        return [(n, m, k, 2, 4) for (n, k) in ((4096, 4096), (11008, 4096), (4096, 11008))
                for m in (64, 128, 256, 512)]
    if name == "decode":
        return [(8192, m, 8192, 3, 8) for m in (1, 8, 16)]
    raise SystemExit(f"unknown workload {name}")


WORKLOAD_DESC = {
    "ffn70b": "BASELINE configs[4]: Llama-2-70B FFN 28672x8192 W2A4, M=4096 tokens",
    "sweep4096": "BASELINE configs[1]: precision sweep W1-4 x A2/A4/A8, M=N=K=4096, 12 GEMMs/step",
    "w2a4_4096": "W2A4 M=N=K=4096",
    "llama7b": "BASELINE configs[2]: Llama-2-7B linear shapes W2A4, M=2048 tokens",
    "llama7b_small": "BASELINE configs[2]: Llama-2-7B linear shapes W2A4, M in {1,16} tokens",
    "llama7b_mid": "BASELINE configs[2]: Llama-2-7B linear shapes W2A4, M in {64,128,256,512}",
    "decode": "BASELINE configs[3]: decode W3A8 K=N=8192, M in {1,8,16}",
}
SHARDED = {"ffn70b"}  # workloads that N-shard one GEMM across the ranks


def ops_of(g):
    n_out, m_tok, k, _, _ = g
    return 2.0 * n_out * m_tok * k


def packed_bytes(rows, k, n):
    return 4 * n * rows * ((k + 31) // 32)


def algorithmic_bytes(g):
    n_out, m_tok, k, nw, nx = g
    return packed_bytes(n_out, k, nw) + packed_bytes(m_tok, k, nx) + 4 * n_out * m_tok


def bench_config(workload: str, world: int) -> dict:
    """The `config` object -- identical in both arms for the same workload and N."""
    gemms = workload_gemms(workload)
    sharded = workload in SHARDED and world > 1
    return {
        "workload": WORKLOAD_DESC[workload],
        "shapes": [list(g) for g in gemms],
        "shape_fields": "[N_out, M_tok, K, n_w, n_x]",
        "gemms_per_step": len(gemms),
        "orientation": "matmul_ap(W[N_out x K,n_w], X[M_tok x K,n_x]) -> int32 [N_out x M_tok]",
        "parallelism": (f"N_out sharded x{world}: contiguous W row blocks, X replicated, "
                        "no data-path collective (all-gather timed separately)" if sharded
                        else ("N-sharded (1 GPU holds all rows)" if workload in SHARDED
                              else f"replicas x{world}: independent GEMMs per GPU")),
    }


def load_json(rel):
    try:
        with open(os.path.join(ROOT, rel)) as f:
            return json.load(f)
    except Exception:
        return {}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 100 ms while the timed region runs (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------- CPU reference arm
class CpuReference:
    """The reference's matmul_ap (oracle/_ref; the C restatement when _ref is absent),
    row-sliced over `threads` host threads, on `rows[i]` W rows of each GEMM of a workload
    (all rows = the full GEMM). Packing is done once, outside the timed calls, as in the
    reference bench (apmm.cpp:163-172)."""

    def __init__(self, gemms, threads: int, budget_s: float | None, seed: int = 1):
        import numpy as np
        from oracle import Oracle, Reference
        self.np = np
        self.threads = threads
        self.kind = "reference" if Reference.available() else "port"
        self.ref = Reference() if self.kind == "reference" else None
        self.orc = Oracle()
        self.gemms = gemms
        rng = np.random.default_rng(seed)
        self.x_planes, self.w_codes = [], []
        for (n_out, m_tok, k, nw, nx) in gemms:
            xc = rng.integers(0, 1 << nx, size=(m_tok, k), dtype=np.uint8)
            self.x_planes.append(self._pack(xc, nx))
            self.w_codes.append(rng.integers(0, 1 << nw, size=(n_out, k), dtype=np.uint8))
        # calibrate the per-W-row cost of each GEMM on a small slice
        cal = max(2 * threads, 32)
        t_row = []
        for i, g in enumerate(gemms):
            r = min(cal, g[0])
            job = self._job(i, r, threads)
            job.run()
            t_row.append(job.run() / r)
        self.t_row = t_row
        full = sum(t * g[0] for t, g in zip(t_row, gemms))
        frac = 1.0 if budget_s is None else min(1.0, budget_s / max(full, 1e-9))
        self.rows = [g[0] if frac >= 1.0 else max(min(g[0], 2 * threads), int(g[0] * frac))
                     for g in gemms]
        self.jobs = [self._job(i, r, threads) for i, r in enumerate(self.rows)]
        self.full = all(r == g[0] for r, g in zip(self.rows, gemms))
        self.sample = ("full GEMMs: " if self.full else "row sample: ") + ", ".join(
            f"{r}/{g[0]} W rows of W{g[3]}A{g[4]} {g[0]}x{g[1]}x{g[2]}"
            for r, g in zip(self.rows, gemms))

    def _pack(self, codes, n):
        return self.ref.pack(codes, n) if self.ref else self.orc.pack(codes, n)

    def _job(self, i, rows, threads):
        n_out, m_tok, k, nw, nx = self.gemms[i]
        wp = self._pack(self.np.ascontiguousarray(self.w_codes[i][:rows]), nw)
        xp = self.x_planes[i]
        if self.ref:
            return self.ref.job(wp, rows, nw, xp, m_tok, nx, k, threads)
        orc = self.orc

        class PortJob:
            def run(self_inner):
                t0 = time.perf_counter()
                orc.matmul_ap_mt(wp, rows, nw, xp, m_tok, nx, k, threads)
                return time.perf_counter() - t0
        return PortJob()

    def step(self) -> tuple[float, float]:
        """One step (every GEMM's sample once); returns (seconds, ops)."""
        secs = sum(j.run() for j in self.jobs)
        ops = sum(r * 2.0 * g[1] * g[2] for r, g in zip(self.rows, self.gemms))
        return secs, ops


def single_thread_figure(gemms, budget_s: float = 6.0) -> dict:
    """The reference as shipped: one thread, warmup 2 + mean of 10 (apmm.cpp:102-109,
    :126-127) on a W-row sample of the first GEMM sized to ~budget_s in total."""
    g = gemms[0]
    import numpy as np
    from oracle import Oracle, Reference
    kind = "reference" if Reference.available() else "port"
    n_out, m_tok, k, nw, nx = g
    rng = np.random.default_rng(2)
    xc = rng.integers(0, 1 << nx, size=(m_tok, k), dtype=np.uint8)
    ref = Reference() if kind == "reference" else None
    orc = Oracle()
    pack = ref.pack if ref else orc.pack
    xp = pack(xc, nx)

    def make(rows):
        wc = rng.integers(0, 1 << nw, size=(rows, k), dtype=np.uint8)
        wp = pack(wc, nw)
        if ref:
            return ref.job(wp, rows, nw, xp, m_tok, nx, k, 1)

        class PortJob:
            def run(self_inner):
                t0 = time.perf_counter()
                orc.matmul_ap_mt(wp, rows, nw, xp, m_tok, nx, k, 1)
                return time.perf_counter() - t0
        return PortJob()
    rows = min(n_out, 4)
    t = make(rows).run()
    rows = int(max(1, min(n_out, rows * (budget_s / 12.0) / max(t, 1e-6))))
    job = make(rows)
    for _ in range(2):
        job.run()
    ts = [job.run() for _ in range(10)]
    mean = sum(ts) / len(ts)
    return {"value": 2.0 * rows * m_tok * k / mean / 1e12, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{rows}/{n_out} W rows of W{nw}A{nx} {n_out}x{m_tok}x{k}, warmup 2 + mean of 10 "
                      "(as shipped, apmm.cpp:102-109)"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    gemms = workload_gemms(args.workload)
    threads = cpu_threads()
    # every step is the full config when that fits ~8 min of CPU for the whole run,
    # otherwise a W-row sample sized to that budget (stated in `sample`)
    budget = 480.0 / max(1, args.steps + args.warmup)
    ref = CpuReference(gemms, threads, None)
    est_full = sum(t * g[0] for t, g in zip(ref.t_row, gemms))
    if est_full > budget:
        ref = CpuReference(gemms, threads, budget)
    for _ in range(args.warmup):
        ref.step()
    secs = ops = 0.0
    for _ in range(args.steps):
        s, o = ref.step()
        secs += s
        ops += o
    tops = ops / secs / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": tops, "unit": UNIT,
        "n_gpus": world if world > 1 else args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.workload in SHARDED else "weak", "vs_baseline": None,
        "dtype": "int32 (bit-plane XOR-popcount, reference CPU kernel)",
        "data": "synthetic (uniform bipolar codes, random_codes semantics)",
        "config": bench_config(args.workload, world if world > 1 else args.gpus),
        "cpu_baseline": {"value": tops, "unit": UNIT, "cores": threads, "kind": ref.kind,
                         "sample": ref.sample, "cpu_model": cpu_model()},
        "e2e": {"value": tops, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["cpu_single_thread"] = single_thread_figure(gemms)
    except Exception as e:
        line["cpu_single_thread"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- parity check
def parity_check(entries, threads):
    """Sampled-row bit-exactness of the Y buffers the timed region produced.

    entries: list of (g, w_planes_dev, x_planes_dev, y_dev). Two W rows per 256-row tile
    (all tiles, all columns) are compared against the reference's matmul_ap (oracle/_ref,
    or the C restatement when _ref is absent) on the same packed inputs."""
    import numpy as np
    import torch
    from oracle import Oracle, Reference
    kind = "reference" if Reference.available() else "port"
    ref = Reference() if kind == "reference" else None
    orc = Oracle()
    gen = np.random.default_rng(7)
    rows_checked = 0
    for (g, wp, xp, y) in entries:
        n_out, m_tok, k, nw, nx = g
        wpr = (k + 31) // 32
        rows = []
        for t0 in range(0, n_out, 256):
            span = min(256, n_out - t0)
            rows.extend(sorted(set(int(t0 + r) for r in gen.integers(0, span, size=2))))
        if n_out - 1 not in rows:
            rows.append(n_out - 1)
        idx = torch.tensor(rows, device=wp.device, dtype=torch.long)
        w_rows = wp.view(nw, n_out, wpr).index_select(1, idx).contiguous().cpu().numpy().view(np.uint32)
        x_h = xp.cpu().numpy().view(np.uint32)
        y_rows = y.index_select(0, idx).cpu().numpy()
        if ref:
            job = ref.job(w_rows.reshape(-1), len(rows), nw, x_h, m_tok, nx, k, threads)
            job.run()
            want = job.result()
        else:
            want = orc.matmul_ap_mt(w_rows.reshape(-1), len(rows), nw, x_h, m_tok, nx, k, threads)
        if not np.array_equal(y_rows, want):
            bad = int((y_rows != want).sum())
            return False, f"MISMATCH: {bad} entries differ in {len(rows)} sampled rows of {g}"
        rows_checked += len(rows)
    return True, (f"ok: {rows_checked} sampled W rows (2 per 256-row tile, all columns) of every "
                  f"timed Y bit-exact vs the {kind} matmul_ap")


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2409_17870_b200 as ap

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = ap.Context(local_rank)
    if args.early_features:  # documented opt-in: this bench's features are static inputs
        ctx.set_early_feature_read(True)
    stream = torch.cuda.Stream(device=dev)  # every launch of the timed region goes here
    torch.cuda.set_stream(stream)
    full_gemms = workload_gemms(args.workload)
    gemms = full_gemms
    sharded = args.workload in SHARDED and world > 1
    if sharded:  # rank p owns W rows [r0, r1) (paper_2409_17870_b200/shard.py)
        from paper_2409_17870_b200.shard import word_shard_bounds as shard_bounds
        n_out, m_tok, k, nw, nx = full_gemms[0]
        r0, r1 = shard_bounds(n_out, world, rank)
        gemms = [(r1 - r0, m_tok, k, nw, nx)]

    # -- synthetic operands: uniform codes (random_codes, verify.cpp:18-22), packed to bit
    #    planes on device (packing excluded from timing, as in apmm.cpp:163-172)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1 + rank)
    ops_step = sum(ops_of(g) for g in gemms)
    # L2 rule: when a step touches less than 2x the 126 MB L2, the inputs (W and X planes)
    # rotate over `nrot` copies (step s uses copy s % nrot), so no step finds them in L2.
    step_bytes = sum(algorithmic_bytes(g) for g in gemms)
    nrot = 1 if step_bytes >= 2 * 126e6 else -(-int(2 * 126e6) // int(step_bytes))
    bufs = []
    for (n_out, m_tok, k, nw, nx) in gemms:
        wpr = (k + 31) // 32
        wps, xps = [], []
        for _ in range(nrot):
            wc = torch.randint(0, 1 << nw, (n_out, k), generator=gen, device=dev, dtype=torch.uint8)
            wp = torch.empty(nw * n_out * wpr, dtype=torch.int32, device=dev)
            ap.cu_pack(wc, n_out, k, nw, wp, ctx)
            wps.append(wp)
            del wc
            xc = torch.randint(0, 1 << nx, (m_tok, k), generator=gen, device=dev, dtype=torch.uint8)
            xp = torch.empty(nx * m_tok * wpr, dtype=torch.int32, device=dev)
            ap.cu_pack(xc, m_tok, k, nx, xp, ctx)
            xps.append(xp)
            del xc
        y = torch.empty((n_out, m_tok), dtype=torch.int32, device=dev)
        bufs.append((wps, xps, y))
    torch.cuda.synchronize()

    def make_step(r):
        def step_r():
            for (g, (wps, xps, y)) in zip(gemms, bufs):
                n_out, m_tok, k, nw, nx = g
                ap.cu_matmul_ap(wps[r], n_out, nw, xps[r], m_tok, nx, k, y, ctx)
        return step_r

    step_fns = [make_step(r) for r in range(nrot)]
    step_i = [0]

    def step():
        step_fns[step_i[0] % nrot]()
        step_i[0] += 1

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # The K timed steps are captured as ONE CUDA graph (the serving pattern: a model step is
    # a chain of these GEMMs) and replayed once in the timed region. The launches keep their
    # programmatic-dependent-launch edges across GEMM boundaries inside the graph, and host
    # launch overhead (Python + C ABI, ~10 us per call) leaves the timed region.
    # --no-graph times the eager launches instead.
    graph = None
    graph_launches = 0
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        n0 = ctx.launch_count()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(args.steps):
                step_fns[i % nrot]()
        graph_launches = (ctx.launch_count() - n0) // args.steps
        torch.cuda.synchronize()

        def step():  # noqa: F811  (heat phase: whole K-step replays)
            graph.replay()
        step()
        torch.cuda.synchronize()
    # heat: ~1 s of untimed steps so clocks settle and the sampler sees the load
    clocks = ClockSampler(local_rank)
    clocks.start()
    t_end = time.time() + (0.0 if args.profile else 1.0)
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()

    # -- timed region: exactly K steps, barrier + synchronize on both sides. No per-kernel
    #    events in here: an event record between two launches would break the programmatic
    #    dependent launch that overlaps the next call's expand with this call's GEMM.
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    if graph is not None:
        graph.replay()  # exactly K steps
        last_rot = (args.steps - 1) % nrot
    else:
        step_i[0] = 0
        for _ in range(args.steps):
            step()
        last_rot = (args.steps - 1) % nrot
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = ctx.launch_count() - launches0
    if graph is not None:  # replays do not pass through the host counter
        launches = graph_launches * args.steps
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # whole-job work per step: the full GEMM when sharded (strong), else every rank's GEMMs
    job_ops_step = sum(ops_of(g) for g in full_gemms) if sharded else world * ops_step
    value = args.steps * job_ops_step / (ms_max * 1e-3) / 1e12

    # -- parity of exactly what was timed (sampled rows vs the reference), before anything
    #    else touches the Y buffers
    parity = None
    if not args.no_parity and not args.profile:
        entries = [(g, wps[last_rot], xps[last_rot], y) for g, (wps, xps, y) in zip(gemms, bufs)]
        ok, msg = parity_check(entries, cpu_threads())
        flag = torch.tensor([0 if ok else 1], dtype=torch.int32, device=dev)
        if world > 1:
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        parity_ok = int(flag.item()) == 0
        parity = msg if (not ok or parity_ok) else "MISMATCH on another rank"


    # -- kernel pass (roofline): the same K steps again with every GEMM / expand launch
    #    bracketed by CUDA events on its launch stream (serialises expand and GEMM). In
    #    graph mode the bracketed steps are captured as a graph too, so the event pairs
    #    time the kernels, not the host's launch gaps.
    ctx.kernel_time(0)
    ctx.kernel_time(1)
    ek0, ek1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.enable_timing(True)
    if graph is not None:
        kgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(kgraph, stream=stream):
            for i in range(args.steps):
                step_fns[i % nrot]()
        ctx.enable_timing(False)
        torch.cuda.synchronize()
        ek0.record(stream)
        kgraph.replay()
        ek1.record(stream)
    else:
        ek0.record(stream)
        for _ in range(args.steps):
            step()
        ek1.record(stream)
    torch.cuda.synchronize()
    ctx.enable_timing(False)
    ms_serial = ek0.elapsed_time(ek1)
    gemm_ms, gemm_n = ctx.kernel_time(0)
    exp_ms, exp_n = ctx.kernel_time(1)

    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_max / args.steps}), flush=True)
        return

    # -- multi-GPU: the all-gather of the N-sharded int32 row blocks (NCCL over NVLink),
    #    timed on its own (compute-only `value` above) and as compute + gather steps
    gather = None
    if sharded:
        n_full, m_full, k, nw, nx = full_gemms[0]
        wpr = (k + 31) // 32
        ms_blk = max(b - a for a, b in (shard_bounds(n_full, world, p) for p in range(world)))
        send = torch.zeros((ms_blk, m_full), dtype=torch.int32, device=dev)
        recv = torch.empty((world * ms_blk, m_full), dtype=torch.int32, device=dev)
        y0 = bufs[0][2]

        def gather_only():
            send[: y0.shape[0]].copy_(y0)
            dist.all_gather_into_tensor(recv, send)

        for _ in range(3):
            gather_only()
        torch.cuda.synchronize()

        def timed(fn):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(args.steps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            tt = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt.item()) / args.steps

        g_ms = timed(gather_only)

        def compute_gather():
            step_fns[0]()
            gather_only()
        cg_ms = timed(compute_gather)
        recv_bytes = (world - 1) * ms_blk * m_full * 4
        gather = {"format": "int32 Y row blocks", "collective": f"all_gather_into_tensor ({dist.get_backend()})",
                  "ms_per_step": g_ms, "recv_bytes_per_rank": recv_bytes,
                  "algbw_GBps": recv_bytes / (g_ms * 1e-3) / 1e9,
                  "compute_plus_gather_ms_per_step": cg_ms,
                  "compute_plus_gather_TOPS": job_ops_step / (cg_ms * 1e-3) / 1e12}
        # the consumer's view: the next layer needs X' = dequant(Y)^T as
        # A4 packed planes. Per rank: GEMM + dequant epilogue (+ per-token absmax), a MAX
        # all-reduce of 4096 doubles, quantize + pack of the rank's word block, all-gather of
        # the packed planes (+ one word-block re-layout) -- instead of the int32 gather.
        from paper_2409_17870_b200.shard import sharded_matmul_requant
        n_next = 4
        wfull = torch.empty(nw * n_full * wpr, dtype=torch.int32, device=dev)
        r0, r1 = shard_bounds(n_full, world, rank)
        wfull.view(nw, n_full, wpr)[:, r0:r1].copy_(bufs[0][0][0].view(nw, r1 - r0, wpr))
        sw_full = torch.rand(n_full, dtype=torch.float64, device=dev, generator=gen) + 0.5
        sx = torch.rand(m_full, dtype=torch.float64, device=dev, generator=gen) + 0.5
        xq = bufs[0][1][0]

        def layer_packed():
            return sharded_matmul_requant(wfull, n_full, nw, sw_full, 1, xq, m_full, nx, sx, 1,
                                          k, n_next, 1)
        for _ in range(2):
            layer_packed()
        torch.cuda.synchronize()
        lp_ms = timed(layer_packed)
        wps_ = -(-n_full // 32)
        packed_recv = (world - 1) * n_next * m_full * (-(-wps_ // world)) * 4
        gather["next_layer_packed"] = {
            "format": f"A{n_next} packed planes of X' = dequant(Y)^T + per-token scales",
            "ms_per_step": lp_ms, "recv_bytes_per_rank": packed_recv,
            "bytes_vs_int32": packed_recv / recv_bytes,
            "note": ("GEMM + dequant/absmax epilogue + absmax all-reduce + requant/pack + packed "
                     "all-gather, per step; W rows split on 32-row word boundaries")}

    # -- single GPU: the layer form the next layer consumes, timed on its
    #    own: GEMM + dequant epilogue with the per-token absmax fused in + requantize/pack of
    #    X' = dequant(Y)^T to A4 planes (apmm_cu_matmul_ap_requant), vs the int32 GEMM above
    requant = None
    if not sharded and args.workload in SHARDED:
        g0 = gemms[0]
        n_out, m_tok, k, nw, nx = g0
        wps, xps, _ = bufs[0]
        sw = torch.rand(n_out, dtype=torch.float64, device=dev, generator=gen) + 0.5
        sx = torch.rand(m_tok, dtype=torch.float64, device=dev, generator=gen) + 0.5
        yf = torch.empty((n_out, m_tok), dtype=torch.float32, device=dev)
        n_next = 4
        nplanes = torch.empty(n_next * m_tok * (-(-n_out // 32)), dtype=torch.int32, device=dev)
        nscales = torch.empty(m_tok, dtype=torch.float64, device=dev)

        def rq_step():
            ap.cu_matmul_ap_requant(wps[0], n_out, nw, sw, 1, xps[0], m_tok, nx, sx, 1, k, n_next,
                                    1, yf, nplanes, nscales, ctx=ctx, stream=stream)
        for _ in range(2):
            rq_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(3, min(args.steps, 10))
        e0.record(stream)
        for _ in range(reps):
            rq_step()
        e1.record(stream)
        torch.cuda.synchronize()
        rq_ms = e0.elapsed_time(e1) / reps
        requant = {"api": "apmm_cu_matmul_ap_requant (W2A4 GEMM -> dequant + absmax -> A4 planes)",
                   "ms_per_step": rq_ms, "TOPS": ops_step / (rq_ms * 1e-3) / 1e12,
                   "out_bytes": int(nplanes.numel() * 4 + nscales.numel() * 8),
                   "out_bytes_int32_Y": int(4 * n_out * m_tok),
                   "note": "eager launches, includes the NonFinite check's stream sync per call"}
        del yf

    # -- e2e through the public host API: pinned host planes -> H2D -> GEMM -> D2H int32
    e2e_steps = max(1, min(args.steps, 3))
    host = []
    h2d = d2h = 0
    for (g, (wps, xps, y)) in zip(gemms, bufs):
        wp, xp = wps[0], xps[0]
        hw = torch.empty(wp.shape, dtype=torch.int32, pin_memory=True)
        hx = torch.empty(xp.shape, dtype=torch.int32, pin_memory=True)
        hy = torch.empty(tuple(y.shape), dtype=torch.int32, pin_memory=True)
        hw.copy_(wp)
        hx.copy_(xp)
        host.append((g, ap.PackedBitPlanes(g[0], g[2], ap.BitWidth(g[3]), hw.numpy().view(np.uint32)),
                     ap.PackedBitPlanes(g[1], g[2], ap.BitWidth(g[4]), hx.numpy().view(np.uint32)),
                     hy))
        h2d += 4 * (wp.numel() + xp.numel())
        d2h += 4 * y.numel()
    lib = ctx.lib
    import ctypes as C

    def e2e_step():
        for (g, pw, px, hy) in host:
            st = lib.apmm_matmul_ap(ctx.h, pw.words().ctypes.data_as(C.c_void_p), g[0], g[3],
                                    px.words().ctypes.data_as(C.c_void_p), g[1], g[4], g[2],
                                    C.c_void_p(hy.data_ptr()))
            if st != 0:
                raise RuntimeError(lib.apmm_last_error().decode())

    e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = e2e_steps * job_ops_step / float(te.item()) / 1e12

    if rank != 0:
        if parity is not None and not parity_ok:
            sys.exit(1)
        return
    peaks = load_json("MEASURED_PEAKS.json")
    traffic = load_json("profiles/traffic.json")
    bf16 = peaks.get("bf16_tflops")
    i8_peak = 2.0 * bf16 if bf16 else 2.0 * 1590.0
    hbm_peak = peaks.get("hbm_gbs") or 7672.0
    gemm_avg_ms = gemm_ms / max(gemm_n, 1)
    bytes_step = sum(algorithmic_bytes(g) for g in gemms)
    # which roofline bounds the dominant kernel: compare the two ideal times per step
    hbm_bound = bytes_step / (hbm_peak * 1e9) > ops_step / (i8_peak * 1e12)
    small = [g[1] for g in gemms]
    kname = ("skinny_kernel (weight planes -> mma.sync u8 fragments)" if max(small) <= 8 else
             "skinny_kernel (M_tok <= 8) / stream_tc_kernel (12 <= M_tok <= 64: weight planes "
             "expanded into TMEM, tcgen05.mma kind::i8 A-from-TMEM)" if max(small) <= 64 else
             "gemm_u8_pair_kernel / gemm_u8_tc_kernel / gemm_pair_wplanes_kernel / "
             "stream_tc_kernel (tcgen05.mma kind::i8)")
    per_rank_step_s = ms_max * 1e-3 / args.steps
    if hbm_bound:
        achieved = (args.steps * bytes_step / max(gemm_n, 1)) / (gemm_avg_ms * 1e-3) / 1e9
        step_achieved = bytes_step / per_rank_step_s / 1e9
        peak, unit = hbm_peak, "GB/s"
        peak_src = ("MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if peaks.get("hbm_gbs")
                    else "B200_PROFILING.md fallback")
    else:
        achieved = (args.steps * ops_step / max(gemm_n, 1)) / (gemm_avg_ms * 1e-3) / 1e12
        step_achieved = ops_step / per_rank_step_s / 1e12
        peak, unit = i8_peak, "TFLOP/s"
        peak_src = ("2 x measured bf16 burst (MEASURED_PEAKS.json bf16_tflops); "
                    "dense i8 = 2x dense bf16 on B200" if bf16 else
                    "2 x fallback bf16 1590 (B200_PROFILING.md)")
    i8_ceiling = (load_json("profiles/i8_mma_peak.json") or {}).get("i8_tops")
    tr_ent = traffic.get(args.workload if not sharded else f"{args.workload}_p{world}") or {}
    tr = tr_ent.get("bytes")  # dram read+write bytes per launch (ncu --set full), or None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.workload in SHARDED else "weak", "vs_baseline": None,
        "dtype": "u8 codes x u8 codes -> s32 (exact int)",
        "data": "synthetic (uniform bipolar codes, packed to bit planes on device)",
        "config": bench_config(args.workload, world),
        "per_rank_shapes": [list(g) for g in gemms],
        "launch": "eager" if graph is None else "one cuda graph of the K timed steps",
        "pdl_feature_reads": ("early (--early-features: features are static inputs here)"
                              if args.early_features else
                              "after the previous kernel (safe default; features may be its output)"),
        "l2": ("no flush: per-step packed inputs %.0f MB + outputs %.0f MB > 2 x 126 MB L2" % (
            sum(packed_bytes(g[0], g[2], g[3]) + packed_bytes(g[1], g[2], g[4]) for g in gemms) / 1e6,
            sum(4 * g[0] * g[1] for g in gemms) / 1e6) if nrot == 1 else
            "W and X planes rotate over %d copies (step s uses copy s %% %d): %.0f MB "
            "between reuses > 2 x 126 MB L2" % (nrot, nrot, nrot * step_bytes / 1e6)),
        "parity": parity,
        "clocks": clk,
        "gpu_launches": int(launches),
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "api": "apmm_matmul_ap (host C ABI, pinned buffers)"},
        "roofline": {"bound": "hbm" if hbm_bound else "tensor", "achieved": achieved,
                     "peak": peak, "unit": unit, "frac": achieved / peak, "traffic": tr,
                     "traffic_source": tr_ent.get("kernel"),
                     "kernel": kname, "peak_source": peak_src,
                     "achieved_step": step_achieved, "frac_step": step_achieved / peak,
                     "frac_note": ("frac = dominant kernel alone (event-timed launches); "
                                   "frac_step = the whole pipelined step (expand + GEMM) per rank; "
                                   "the north-star 60% target is read against `peak`"),
                     "i8_mma_ceiling_tops": None if hbm_bound else i8_ceiling,
                     "frac_of_i8_mma_ceiling": (achieved / i8_ceiling
                                                if (i8_ceiling and not hbm_bound) else None),
                     "frac_step_of_i8_mma_ceiling": (step_achieved / i8_ceiling
                                                     if (i8_ceiling and not hbm_bound) else None),
                     "i8_mma_ceiling_source": None if hbm_bound else
                         "profiles/i8_mma_peak.json: this pair kernel with operand reloads off, 8192^3",
                     "algorithmic_bytes_per_step": bytes_step,
                     "algorithmic_ops_per_step": ops_step,
                     "gemm_us_avg": 1e3 * gemm_avg_ms,
                     "expand_us_avg": 1e3 * exp_ms / max(exp_n, 1),
                     "serialized_ms_per_step": ms_serial / args.steps,
                     "gemm_share_of_serialized_step": gemm_ms / ms_serial,
                     "expand_share_of_serialized_step": exp_ms / ms_serial},
    }
    if gather is not None:
        line["gather"] = gather
    if requant is not None:
        line["next_layer_requant"] = requant
    if world == 1 and not args.no_cpu_baseline:
        try:
            ref = CpuReference(gemms, cpu_threads(), 10.0)
            s, o = ref.step()
            line["cpu_baseline"] = {"value": o / s / 1e12, "unit": UNIT, "cores": ref.threads,
                                    "kind": ref.kind, "sample": ref.sample,
                                    "cpu_model": cpu_model()}
        except Exception as e:  # the baseline must never hide the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if parity is not None and not parity_ok:
        sys.exit(1)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap_ = argparse.ArgumentParser()
    ap_.add_argument("--gpus", type=int, default=1)
    ap_.add_argument("--steps", type=int, default=20)
    ap_.add_argument("--warmup", type=int, default=3)
    ap_.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap_.add_argument("--workload", default="ffn70b", choices=list(WORKLOAD_DESC))
    ap_.add_argument("--no-cpu-baseline", action="store_true")
    ap_.add_argument("--no-parity", action="store_true",
                     help="skip the post-timing sampled-row parity check (dev only)")
    ap_.add_argument("--no-graph", action="store_true",
                     help="time eager launches instead of replaying the step as a CUDA graph")
    ap_.add_argument("--early-features", action="store_true",
                     help="APMM_OPT_EARLY_FEATURE_READ: let the next call read its (static) "
                          "features while the previous GEMM drains (not the default)")
    ap_.add_argument("--profile", action="store_true",
                     help="for ncu: no heat phase, no e2e, no CPU baseline (numbers invalid)")
    args = ap_.parse_args()
    args.warmup = max(3, args.warmup)

    in_torchrun = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not in_torchrun and args.impl == "ours":
        # one process per GPU: re-launch under torch.distributed.run (127.0.0.1 rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if in_torchrun and args.gpus not in (1, world):
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # APMM_BENCH_BACKEND=gloo (dev): exercise the multi-rank code path with several ranks
        # sharing the GPUs that exist (NCCL needs one GPU per rank); numbers are not valid
        backend = os.environ.get("APMM_BENCH_BACKEND", "nccl")
        local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
