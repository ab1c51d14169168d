"""SASS instruction census of the shipped libmorap_cuda.so (profiles/r02_sass_counts.txt):
per kernel, TMA bulk copies (UBLKCP), mbarrier ops (SYNCS), and DFMA -- which must be 0 for
bitwise parity with the reference (no FMA contraction).  python scripts/sass_census.py > out.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2305_04397_b200", "libmorap_cuda.so")
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
keys = ["UBLKCP", "SYNCS", "DFMA", "DMUL", "DADD", "LDS", "LDG", "STG", "ATOMG", "REDG", "BAR.SYNC", "SHFL"]
rows, tot = [], collections.Counter()
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    m = re.search(r"::(k_[A-Za-z_0-9]+(<[^>]*>)?)\(", d)
    short = (m.group(1) if m else d[:40]).replace("<(bool)0>", "<false>").replace("<(bool)1>", "<true>")
    c = collections.Counter()
    for line in f.split("\n"):
        mm = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if not mm:
            continue
        op = mm.group(2)
        for k in keys:
            if op == k or op.startswith(k + "."):
                c[k] += 1
    rows.append((short, c))
    tot.update(c)
print("SASS instruction counts per kernel of the shipped libmorap_cuda.so (sm_100a cubin), scripts/sass_census.py")
print("UBLKCP = cp.async.bulk (TMA 1-D bulk copies), SYNCS = mbarrier ops; DFMA must be 0 (bitwise parity with the "
      "reference: no FMA contraction).")
print(f"{'kernel':36s}" + "".join(f"{k:>9s}" for k in keys))
for n, c in sorted(rows):
    print(f"{n:36s}" + "".join(f"{c[k]:9d}" for k in keys))
print(f"total DFMA in the library: {tot['DFMA']}; UBLKCP: {tot['UBLKCP']}; SYNCS: {tot['SYNCS']}")
