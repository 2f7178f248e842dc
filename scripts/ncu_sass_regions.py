"""Stall-reason samples and executed instructions of an ncu report, split into the row loops of the
decode kernel (found statically, as scripts/sass_loops.py does) and the rest.
usage: python scripts/ncu_sass_regions.py report.ncu-rep [LIB.so] [kernel-substring]"""
import collections
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_loops import functions, row_loops  # noqa: E402

rep = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2208_08711_b200/libl3_b200.so"
pat = sys.argv[3] if len(sys.argv) > 3 else "l3_decode_kernelILb1ELb0ELb0ELb0E"
fs = functions(lib)
name = [n for n in fs if pat in n][0]
loops = [(t, a) for t, a, _ in row_loops(fs[name])]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
recs = list(csv.reader(io.StringIO(out)))
hdr = recs[1]
base = None
agg = collections.defaultdict(collections.Counter)
for r in recs[2:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    addr = int(d["Address"], 16)
    if base is None:
        base = addr
    off = addr - base
    region = "other"
    for i, (t, a) in enumerate(loops):
        if t <= off <= a:
            region = f"loop{i}@{t:#x}"
    c = agg[region]
    c["inst"] += int(d["Instructions Executed"] or 0)
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            c[k] += int(d[k] or 0)
for reg, c in agg.items():
    tot = sum(v for k, v in c.items() if k.startswith("stall_"))
    print(reg, "inst", c["inst"], "samples", tot)
    print("   ", ", ".join(f"{k[6:]} {v}" for k, v in c.most_common() if k.startswith("stall_") and v))
