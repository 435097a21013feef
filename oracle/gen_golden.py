"""TEST INFRASTRUCTURE: generate tests/golden/reference_vectors.json by running the
reference itself (oracle/_ref/libapmm_ref.so, compiled from /root/reference/proj/src).

    python oracle/gen_golden.py

The fixture pins the C restatement (apmm_oracle.c) and the GPU path to the reference's
own outputs on inputs the GPU box can replay without /root/reference present.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import PER_ROW, PER_TENSOR, Reference, build  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "reference_vectors.json")


def hexd(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).reshape(-1)]


def main():
    build()
    ref = Reference()
    rng = np.random.default_rng(20240917)
    doc = {"generator": "oracle/gen_golden.py via oracle/_ref/libapmm_ref.so (reference proj/src)",
           "rng": {}, "pack": [], "quantize": [], "matmul": [], "plane_products": []}
    for seed in (1, 42, 99, 5489):
        doc["rng"][str(seed)] = [str(int(v)) for v in ref.rng_draws(seed, 16)]
    # pack / unpack
    for (rows, cols, n) in [(1, 1, 1), (1, 33, 1), (2, 2, 2), (3, 70, 5), (5, 45, 3), (4, 64, 8)]:
        codes = rng.integers(0, 1 << n, size=(rows, cols), dtype=np.uint8)
        words = ref.pack(codes, n)
        doc["pack"].append({"rows": rows, "cols": cols, "n": n, "codes": codes.reshape(-1).tolist(),
                            "words": words.tolist()})
    # quantize (fp64, hex-exact)
    for (rows, cols, n, gran, zero_row) in [(1, 4, 2, PER_TENSOR, False), (3, 7, 3, PER_ROW, True),
                                            (5, 9, 8, PER_TENSOR, False), (4, 33, 1, PER_ROW, False),
                                            (6, 40, 4, PER_ROW, False), (2, 5, 6, PER_TENSOR, True)]:
        x = rng.uniform(-100.0, 100.0, size=(rows, cols))
        x[rng.random(size=x.shape) < 0.1] = 0.0
        if zero_row:
            x[0, :] = 0.0
        codes, scales = ref.quantize(x, n, gran)
        doc["quantize"].append({"rows": rows, "cols": cols, "n": n, "gran": gran, "x": hexd(x),
                                "codes": codes.reshape(-1).tolist(), "scales": hexd(scales)})
    # matmul_ap: random shapes incl. ragged K, all widths, the admissible W8A8 edge
    shapes = [(1, 1, 1, 1, 1), (6, 5, 40, 3, 2), (7, 9, 33, 8, 8), (17, 3, 95, 4, 1),
              (32, 32, 200, 2, 2), (13, 31, 129, 5, 7), (64, 40, 300, 1, 8), (3, 3, 1, 8, 8),
              (9, 11, 257, 6, 3), (2, 2, 33025, 8, 8)]
    for (m, n_, k, nw, nx) in shapes:
        wc = rng.integers(0, 1 << nw, size=(m, k), dtype=np.uint8)
        xc = rng.integers(0, 1 << nx, size=(n_, k), dtype=np.uint8)
        wp, xp = ref.pack(wc, nw), ref.pack(xc, nx)
        y = ref.matmul_ap(wp, m, nw, xp, n_, nx, k)
        doc["matmul"].append({"rows_w": m, "rows_x": n_, "k": k, "n_w": nw, "n_x": nx,
                              "w_words": wp.tolist(), "x_words": xp.tolist(),
                              "y": y.reshape(-1).tolist()})
    # plane-product stack of the 2-bit worked example (test_kernel.cpp:125-136)
    wc = np.array([[0b11, 0b10]], dtype=np.uint8)  # values [3, 1]
    xc = np.array([[0b01, 0b11]], dtype=np.uint8)  # values [-1, 3]
    stack, y = ref.plane_products(ref.pack(wc, 2), 1, 2, ref.pack(xc, 2), 1, 2, 2)
    doc["plane_products"].append({"w_codes": wc.reshape(-1).tolist(), "x_codes": xc.reshape(-1).tolist(),
                                  "n_w": 2, "n_x": 2, "k": 2, "stack": stack.reshape(-1).tolist(),
                                  "y": y.reshape(-1).tolist()})
    # APMM v1 tensor files written by the reference's serializer (tensor_file.cpp:135-157):
    # the 1x4 W2 golden of test_tensor_file.cpp:21-26, a per-row W3 5x37 tensor (ragged
    # words), a per-tensor W4 3x64 one and a float32 2x3 tensor; stored as files next to the
    # JSON so the GPU box can upload them with no reference present.
    gdir = os.path.dirname(OUT)
    files = []
    for name, x, n, gran in [("w2_1x4_tensor", np.array([[3.0, -1.0, 1.0, -3.0]]), 2, PER_TENSOR),
                             ("w3_5x37_row", rng.uniform(-8, 8, size=(5, 37)), 3, PER_ROW),
                             ("w4_3x64_tensor", rng.uniform(-2, 2, size=(3, 64)), 4, PER_TENSOR)]:
        data = ref.serialize_quantized(x, n, gran)
        codes, scales = ref.quantize(x, n, gran)
        with open(os.path.join(gdir, name + ".apmm"), "wb") as f:
            f.write(data)
        files.append({"file": name + ".apmm", "kind": 1, "rows": x.shape[0], "cols": x.shape[1],
                      "n": n, "gran": gran, "words": ref.pack(codes, n).tolist(),
                      "scales": hexd(scales)})
    xf = np.array([[0.5, -1.25, 3.0], [1e10, -7.5e-3, 0.0]])  # test_tensor_file.cpp:56
    with open(os.path.join(gdir, "f32_2x3.apmm"), "wb") as f:
        f.write(ref.serialize_float(xf))
    files.append({"file": "f32_2x3.apmm", "kind": 0, "rows": 2, "cols": 3,
                  "values": hexd(xf.astype(np.float32).astype(np.float64))})
    doc["tensor_files"] = files
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
