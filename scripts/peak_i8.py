"""Measure the dense int8 tensor throughput of cuBLAS on this B200 (torch._int_mm, s8 x s8 -> s32)
as a library reference for the i8 roofline denominator. Writes profiles/i8_peak.json."""
import json, os, sys, time, torch
dev = torch.device("cuda")
res = {}
for n in (4096, 8192, 16384):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"cublas_int_mm_{n}"] = {"ms": best, "tops": 2 * n**3 / best / 1e9}
    # sustained: back to back 2 s
    t_end = time.time() + 2.0; iters = 0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() < t_end:
        for _ in range(10): torch._int_mm(a, b)
        iters += 10
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    res[f"cublas_int_mm_{n}"]["sustained_tops"] = 2 * n**3 * iters / e0.elapsed_time(e1) / 1e9
print(json.dumps(res, indent=1))
os.makedirs("profiles", exist_ok=True)
json.dump(res, open("gpurun_out/i8_peak.json", "w"), indent=1)
