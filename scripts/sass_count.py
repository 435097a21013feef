"""Static SASS opcode histogram of one kernel in libapmm_b200.so (dev tool):
    python scripts/sass_count.py <substring of mangled name> [lib]"""
import collections
import re
import subprocess
import sys

pat = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2409_17870_b200/libapmm_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if pat not in name:
        continue
    ops = collections.Counter()
    lines = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", f)
    imma = [i for i, l in enumerate(lines) if "IMMA" in l]
    body = lines[imma[0] - 150: imma[-1] + 20] if imma else lines
    for l in body:
        tok = l.split()
        op = tok[1] if tok and tok[0].startswith("@") else (tok[0] if tok else "")
        ops[op.split(".")[0]] += 1
    print(name[:80], "total", len(lines), "loop-ish", len(body))
    print("  ", ops.most_common(14))
