"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel: count, mean, share."""
import collections, csv, io, sys

def load(path):
    text = open(path).read()
    i = text.find('"ID"')
    return list(csv.DictReader(io.StringIO(text[i:])))

def short(name):
    n = name.replace("void ", "")
    for tok in ("gemm_u8_tc_kernel", "expand_kernel", "pack_kernel", "unpack_kernel", "quantize",
                "distribution_elementwise", "absmax_kernel", "gemv", "splitk"):
        if tok in n:
            return tok
    return n.split("(")[0][-40:]

if __name__ == "__main__":
    rows = load(sys.argv[1])
    skip = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else {"distribution_elementwise", "pack_kernel"}
    agg = collections.OrderedDict()
    for r in rows:
        k = short(r["Kernel Name"])
        if k in skip:
            continue
        agg.setdefault(k, []).append(float(r["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'mean_us':>9s} {'min_us':>8s} {'total_us':>10s} {'share':>6s}")
    for k, v in agg.items():
        print(f"{k:28s} {len(v):8d} {sum(v)/len(v):9.2f} {min(v):8.2f} {sum(v):10.1f} {sum(v)/tot:6.1%}")
