#!/usr/bin/env python3
"""Benchmark of the B200 bipolar-INT WnAm GEMM (arXiv 2409.17870 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload sweep4096|w2a4_4096|llama7b|decode|ffn70b]

Default workload = BASELINE.json configs[1]: the precision sweep W1..W4 x A2/A4/A8 at
M=N=K=4096 on one B200. One step = the 12 GEMMs of the sweep, each the full hot path
through the C ABI (apmm_cu_matmul_ap: packed bit planes in HBM -> int32 Y in HBM).
Metric = effective TOPS = sum(2*M*N*K) / device time (BASELINE.json `metric`).

Multi-GPU (torchrun, one process per GPU): every rank runs the same per-GPU sweep on its
own GPU (independent GEMMs; no data-path collective) -> "scaling": "weak"; the reported
value is all ranks' work / max-over-ranks device time.

`--impl reference` times the reference's own CPU matmul_ap (oracle/_ref, compiled from
/root/reference/proj/src), row-sliced over all host threads, on a bounded row sample of the
same workload; only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ----------------------------------------------------------------------------- workloads
SWEEP_BITS = [(nw, nx) for nw in (1, 2, 3, 4) for nx in (2, 4, 8)]


def workload_gemms(name: str):
    """List of (rows_w=N_out, rows_x=M_tok, K, n_w, n_x) in reference orientation
    matmul_ap(W[N_out x K], X[M_tok x K]) -> Y[N_out x M_tok]."""
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
    if name == "decode":
        return [(8192, m, 8192, 3, 8) for m in (1, 8, 16)]
    if name == "ffn70b":
        return [(28672, 4096, 8192, 2, 4)]
    raise SystemExit(f"unknown workload {name}")


WORKLOAD_DESC = {
    "sweep4096": "BASELINE configs[1]: precision sweep W1-4 x A2/A4/A8, M=N=K=4096, 12 GEMMs/step",
    "w2a4_4096": "W2A4 M=N=K=4096",
    "llama7b": "BASELINE configs[2]: Llama-2-7B linear shapes W2A4, M=2048 tokens",
    "decode": "BASELINE configs[3]: decode W3A8 K=N=8192, M in {1,8,16}",
    "llama7b_small": "BASELINE configs[3]: Llama-2-7B linear shapes W2A4, M in {1,16} tokens",
    "ffn70b": "BASELINE configs[4]: Llama-2-70B FFN 28672x8192 W2A4, M=4096",
}


def ops_of(g):
    n_out, m_tok, k, _, _ = g
    return 2.0 * n_out * m_tok * k


def packed_bytes(rows, k, n):
    return 4 * n * rows * ((k + 31) // 32)


def algorithmic_bytes(g):
    n_out, m_tok, k, nw, nx = g
    return packed_bytes(n_out, k, nw) + packed_bytes(m_tok, k, nx) + 4 * n_out * m_tok


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


def load_i8_ceiling():
    """The pair GEMM's own tcgen05 kind::i8 ceiling (scripts/i8_mma_peak.py: the real kernel
    with operand reloads switched off), reported beside the contract's peak."""
    p = os.path.join(ROOT, "profiles", "i8_mma_peak.json")
    try:
        with open(p) as f:
            return json.load(f).get("i8_tops")
    except Exception:
        return None


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


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
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class CpuReference:
    """The reference's matmul_ap (oracle/_ref) -- or the C restatement when _ref is absent --
    row-sliced over all host threads, on a row sample of each GEMM of the workload."""

    def __init__(self, gemms, budget_s: float, threads: int):
        import numpy as np
        from oracle import Oracle, Reference
        self.np = np
        self.threads = threads
        self.kind = "reference" if Reference.available() else "port"
        self.ref = Reference() if self.kind == "reference" else None
        self.orc = Oracle()
        rng = np.random.default_rng(1)
        self.full = gemms
        # calibrate: per-row cost of each GEMM at a small sample
        self.ops_per_row = [2.0 * g[1] * g[2] for g in gemms]
        cal_rows = max(2 * threads, 32)
        self.inputs = []
        for (n_out, m_tok, k, nw, nx) in gemms:
            wc = rng.integers(0, 1 << nw, size=(min(n_out, 4096), k), dtype=np.uint8)
            xc = rng.integers(0, 1 << nx, size=(m_tok, k), dtype=np.uint8)
            self.inputs.append((wc, xc, nw, nx, k))
        t_row = []
        for i, g in enumerate(gemms):
            job = self._job(i, min(cal_rows, g[0]))
            job.run()
            dt = job.run()
            t_row.append(dt / min(cal_rows, g[0]))
        per_step_full = sum(t * g[0] for t, g in zip(t_row, gemms))
        frac = min(1.0, budget_s / max(per_step_full, 1e-9))
        self.rows = [max(min(g[0], 4096), 1) for g in gemms]
        self.rows = [max(min(r, int(round(g[0] * frac))), min(g[0], 2 * threads))
                     for r, g in zip(self.rows, gemms)]
        self.jobs = [self._job(i, r) for i, r in enumerate(self.rows)]
        self.sample = ", ".join(f"{r}/{g[0]} W rows of W{g[3]}A{g[4]} {g[0]}x{g[1]}x{g[2]}"
                                for r, g in zip(self.rows, gemms))

    def _job(self, i, rows):
        wc, xc, nw, nx, k = self.inputs[i]
        wcs = self.np.ascontiguousarray(wc[:rows])
        if self.kind == "reference":
            wp = self.ref.pack(wcs, nw)
            xp = self.ref.pack(xc, nx)
            return self.ref.job(wp, rows, nw, xp, xc.shape[0], nx, k, self.threads)
        wp = self.orc.pack(wcs, nw)
        xp = self.orc.pack(xc, nx)
        orc, th, mx = self.orc, self.threads, xc.shape[0]

        class PortJob:
            def run(self_inner):
                t0 = time.perf_counter()
                orc.matmul_ap_mt(wp, rows, nw, xp, mx, nx, k, th)
                return time.perf_counter() - t0
        return PortJob()

    def step(self) -> tuple[float, float]:
        """Run one sample step; returns (seconds, ops)."""
        secs = sum(j.run() for j in self.jobs)
        ops = sum(r * opr for r, opr in zip(self.rows, self.ops_per_row))
        return secs, ops


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    gemms = workload_gemms(args.workload)
    threads = cpu_threads()
    budget = max(0.5, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    ref = CpuReference(gemms, budget, threads)
    for _ in range(args.warmup):
        ref.step()
    secs = ops = 0.0
    for _ in range(args.steps):
        s, o = ref.step()
        secs += s
        ops += o
    tops = ops / secs / 1e12
    line = {
        "impl": "reference", "metric": "effective TOPS (2MNK/s)", "value": tops, "unit": "TOPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32 (bit-plane XOR-popcount)", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[args.workload], "gemms": len(gemms),
                   "orientation": "matmul_ap(W[N_out x K], X[M_tok x K])"},
        "cpu_baseline": {"value": tops, "unit": "TOPS", "cores": threads, "kind": ref.kind,
                         "sample": ref.sample},
        "e2e": {"value": tops, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2409_17870_b200 as ap

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = ap.Context(local_rank)
    stream = torch.cuda.Stream(device=dev)  # every launch of the timed region goes here
    torch.cuda.set_stream(stream)
    gemms = workload_gemms(args.workload)
    # configs[4] (70B FFN): N_out sharded across the ranks (contiguous row blocks of W, X
    # replicated; paper_2409_17870_b200/shard.py) -> strong scaling of one GEMM, optionally
    # followed by the NCCL all-gather of the int32 row blocks (--gather). Every other
    # workload runs the same per-GPU GEMMs on each rank (weak scaling, no collective).
    sharded = args.workload == "ffn70b" and world > 1
    full_gemms = gemms
    if sharded:
        from paper_2409_17870_b200.shard import shard_bounds
        n_out, m_tok, k, nw, nx = gemms[0]
        r0, r1 = shard_bounds(n_out, world, rank)
        gemms = [(r1 - r0, m_tok, k, nw, nx)]

    # -- synthetic operands: uniform codes (like random_codes, verify.cpp:18-22), packed to
    #    bit planes on device (packing excluded from timing, as in apmm.cpp:163-172)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1 + rank)
    ops_step = sum(ops_of(g) for g in gemms)
    # L2 rule: when a step touches less than 2x the 126 MB L2, the weight planes rotate over
    # `nrot` copies (step s uses copy s % nrot), so no step finds its weights in L2.
    step_bytes = sum(packed_bytes(g[0], g[2], g[3]) + packed_bytes(g[1], g[2], g[4]) +
                     4 * g[0] * g[1] for g in gemms)
    nrot = max(1, -(-int(2 * 126e6) // int(step_bytes))) if step_bytes < 2 * 126e6 else 1
    bufs = []
    for (n_out, m_tok, k, nw, nx) in gemms:
        wpr = (k + 31) // 32
        wps = []
        for _ in range(nrot):
            wc = torch.randint(0, 1 << nw, (n_out, k), generator=gen, device=dev, dtype=torch.uint8)
            wp = torch.empty(nw * n_out * wpr, dtype=torch.int32, device=dev)
            ap.cu_pack(wc, n_out, k, nw, wp, ctx)
            wps.append(wp)
            del wc
        xc = torch.randint(0, 1 << nx, (m_tok, k), generator=gen, device=dev, dtype=torch.uint8)
        xp = torch.empty(nx * m_tok * wpr, dtype=torch.int32, device=dev)
        ap.cu_pack(xc, m_tok, k, nx, xp, ctx)
        y = torch.empty((n_out, m_tok), dtype=torch.int32, device=dev)
        bufs.append((wps, xp, y))
        del xc
    torch.cuda.synchronize()
    gather_out = None
    if sharded and args.gather:
        from paper_2409_17870_b200.shard import max_shard
        n_full, m_full = full_gemms[0][0], full_gemms[0][1]
        gather_send = torch.zeros((max_shard(n_full, world), m_full), dtype=torch.int32, device=dev)
        gather_out = torch.empty((world * gather_send.shape[0], m_full), dtype=torch.int32, device=dev)

    def make_step(r):
        def step_r():
            for (g, (wps, xp, y)) in zip(gemms, bufs):
                n_out, m_tok, k, nw, nx = g
                ap.cu_matmul_ap(wps[r], n_out, nw, xp, m_tok, nx, k, y, ctx)
            if gather_out is not None:  # full N_out x M_tok on every rank (NCCL over NVLink)
                y = bufs[0][2]
                gather_send[: y.shape[0]].copy_(y)
                dist.all_gather_into_tensor(gather_out, gather_send)
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
    eager_step = step
    run_timed = None
    if not args.no_graph and gather_out is None:
        graph = torch.cuda.CUDAGraph()
        n0 = ctx.launch_count()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(args.steps):
                step_fns[i % nrot]()
        graph_launches = (ctx.launch_count() - n0) // args.steps
        torch.cuda.synchronize()

        def run_timed():
            graph.replay()

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
    if run_timed is not None:
        run_timed()  # exactly K steps (one replay of the K-step graph)
    else:
        for _ in range(args.steps):
            step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = ctx.launch_count() - launches0
    if graph is not None:  # replays do not pass through the host counter
        launches = graph_launches * args.steps
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    # -- kernel pass (roofline): the same K steps again with every GEMM / expand launch
    #    bracketed by CUDA events on its launch stream (serialises expand and GEMM). In
    #    graph mode the bracketed steps are captured as a graph too, so the event pairs
    #    time the kernels, not the host's launch gaps (decode kernels are shorter than the
    #    ~10 us Python + C ABI call).
    ctx.kernel_time(0)
    ctx.kernel_time(1)
    ek0, ek1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph is not None:
        ctx.enable_timing(True)
        kgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(kgraph, stream=stream):
            for i in range(args.steps):
                step_fns[i % nrot]()
        ctx.enable_timing(False)
        torch.cuda.synchronize()
        ek0.record(stream)
        kgraph.replay()
        ek1.record(stream)
        torch.cuda.synchronize()
    else:
        ctx.enable_timing(True)
        ek0.record(stream)
        for _ in range(args.steps):
            step()
        ek1.record(stream)
        torch.cuda.synchronize()
        ctx.enable_timing(False)
    ms_serial = ek0.elapsed_time(ek1)
    gemm_ms, gemm_n = ctx.kernel_time(0)
    exp_ms, exp_n = ctx.kernel_time(1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # whole-job work per step: the full GEMM when sharded (strong), else every rank's GEMMs
    job_ops_step = sum(ops_of(g) for g in full_gemms) if sharded else world * ops_step
    value = args.steps * job_ops_step / (ms_max * 1e-3) / 1e12

    # -- e2e through the public host API: pinned host planes -> H2D -> GEMM -> D2H int32
    if args.profile:
        print(json.dumps({"profile_run": True, "ms_per_step": ms_max / args.steps}), flush=True)
        return
    e2e_steps = max(1, min(args.steps, 3))
    host = []
    h2d = d2h = 0
    for (g, (wps, xp, y)) in zip(gemms, bufs):
        wp = wps[0]
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
        return
    peaks = load_peaks()
    traffic = load_traffic()
    bf16 = peaks.get("bf16_tflops")
    i8_peak = 2.0 * bf16 if bf16 else 2.0 * 1590.0
    hbm_peak = peaks.get("hbm_gbs") or 7672.0
    gemm_avg_ms = gemm_ms / max(gemm_n, 1)
    bytes_step = sum(algorithmic_bytes(g) for g in gemms)
    # which roofline bounds the dominant kernel: compare the two ideal times per step
    hbm_bound = bytes_step / (hbm_peak * 1e9) > ops_step / (i8_peak * 1e12)
    skinny = all(g[1] <= 64 for g in gemms)
    kname = ("skinny_kernel (weight planes -> mma.sync u8 fragments)" if skinny else
             "gemm_u8_pair_kernel / gemm_u8_tc_kernel (tcgen05.mma kind::i8)")
    if hbm_bound:
        achieved = (args.steps * bytes_step / max(gemm_n, 1)) / (gemm_avg_ms * 1e-3) / 1e9
        peak, unit = hbm_peak, "GB/s"
        peak_src = ("MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if peaks.get("hbm_gbs")
                    else "B200_PROFILING.md fallback")
    else:
        achieved = (args.steps * ops_step / max(gemm_n, 1)) / (gemm_avg_ms * 1e-3) / 1e12
        peak, unit = i8_peak, "TFLOP/s"
        peak_src = ("2 x measured bf16 burst (MEASURED_PEAKS.json bf16_tflops); "
                    "dense i8 = 2x dense bf16 on B200" if bf16 else
                    "2 x fallback bf16 1590 (B200_PROFILING.md)")
    i8_ceiling = load_i8_ceiling()
    tr_ent = traffic.get(args.workload) or {}
    tr = tr_ent.get("bytes")  # dram read+write bytes per launch (ncu --set full), or None
    line = {
        "metric": "effective TOPS (2MNK/s) of WnAm bipolar-INT GEMM",
        "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None,
        "dtype": "u8 codes x u8 codes -> s32 (exact int)",
        "data": "synthetic (uniform bipolar codes, packed to bit planes on device)",
        "config": {"workload": WORKLOAD_DESC[args.workload], "gemms_per_step": len(gemms),
                   "shapes": [list(g) for g in gemms],
                   "orientation": "matmul_ap(W[N_out x K,n_w], X[M_tok x K,n_x]) -> int32 [N_out x M_tok]",
                   "parallelism": (f"N_out sharded x{world} (row blocks of W, X replicated)"
                                   + (", NCCL all-gather of Y in the step" if gather_out is not None else "")
                                   if sharded else f"replicas x{world} (N-independent GEMMs per GPU)"),
                   "launch": "eager" if graph is None else "one cuda graph of the K timed steps",
                   "l2": ("no flush: per-step packed inputs %.0f MB + outputs %.0f MB > 2 x 126 MB L2" % (
                       sum(packed_bytes(g[0], g[2], g[3]) + packed_bytes(g[1], g[2], g[4]) for g in gemms) / 1e6,
                       sum(4 * g[0] * g[1] for g in gemms) / 1e6) if nrot == 1 else
                       "weight planes rotate over %d copies (step s uses copy s %% %d): %.0f MB "
                       "between reuses > 2 x 126 MB L2" % (nrot, nrot, nrot * step_bytes / 1e6))},
        "clocks": clk,
        "gpu_launches": int(launches),
        "e2e": {"value": e2e_val, "unit": "TOPS", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "api": "apmm_matmul_ap (host C ABI, pinned buffers)"},
        "roofline": {"bound": "hbm" if hbm_bound else "tensor", "achieved": achieved,
                     "peak": peak, "unit": unit, "frac": achieved / peak, "traffic": tr,
                     "traffic_source": tr_ent.get("kernel"),
                     "i8_mma_ceiling_tops": None if hbm_bound else i8_ceiling,
                     "frac_of_i8_mma_ceiling": (achieved / i8_ceiling
                                                if (i8_ceiling and not hbm_bound) else None),
                     "i8_mma_ceiling_source": None if hbm_bound else
                         "profiles/i8_mma_peak.json: this pair kernel with operand reloads off, 8192^3",
                     "kernel": kname, "peak_source": peak_src,
                     "algorithmic_bytes_per_step": bytes_step,
                     "algorithmic_ops_per_step": ops_step,
                     "gemm_us_avg": 1e3 * gemm_avg_ms,
                     "expand_us_avg": 1e3 * exp_ms / max(exp_n, 1),
                     "serialized_ms_per_step": ms_serial / args.steps,
                     "gemm_share_of_serialized_step": gemm_ms / ms_serial,
                     "expand_share_of_serialized_step": exp_ms / ms_serial},
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            ref = CpuReference(gemms, 8.0, cpu_threads())
            s, o = ref.step()
            line["cpu_baseline"] = {"value": o / s / 1e12, "unit": "TOPS", "cores": ref.threads,
                                    "kind": ref.kind, "sample": ref.sample}
        except Exception as e:  # the baseline must never hide the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)


def main():
    ap_ = argparse.ArgumentParser()
    ap_.add_argument("--gpus", type=int, default=1)
    ap_.add_argument("--steps", type=int, default=20)
    ap_.add_argument("--warmup", type=int, default=3)
    ap_.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap_.add_argument("--workload", default="sweep4096",
                     choices=list(WORKLOAD_DESC))
    ap_.add_argument("--no-cpu-baseline", action="store_true")
    ap_.add_argument("--gather", action="store_true",
                     help="ffn70b under torchrun: all-gather the N-sharded Y (NCCL) inside each step")
    ap_.add_argument("--no-graph", action="store_true",
                     help="time eager launches instead of replaying the step as a CUDA graph")
    ap_.add_argument("--profile", action="store_true",
                     help="for ncu: no heat phase, no e2e, no CPU baseline (numbers invalid)")
    args = ap_.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
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
