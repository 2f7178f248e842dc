"""Executed SASS of an ncu report, per warp-row: every instruction executed at least FRAC times per
decoded (unit, row), in address order, with its stall samples. Shows the dynamic hot path of the row
loop, which static counts (scripts/sass_loops.py) mix with the inlined slow paths.
usage: python scripts/ncu_sass_hot.py report.ncu-rep WARP_ROWS [FRAC=0.2]
(WARP_ROWS: C3 = 12288 units x 128 rows = 1572864)"""
import csv
import io
import subprocess
import sys

rep, wr = sys.argv[1], float(sys.argv[2])
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.2
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
recs = list(csv.reader(io.StringIO(out)))
hdr = recs[1]
rows = [dict(zip(hdr, r)) for r in recs[2:] if len(r) == len(hdr)]
tot = sum(int(r["Instructions Executed"] or 0) for r in rows)
hot = [r for r in rows if int(r["Instructions Executed"] or 0) > frac * wr]
print(f"total {tot} = {tot / wr:.1f} per warp-row; {len(hot)} instructions above {frac}/row = "
      f"{sum(int(r['Instructions Executed']) for r in hot) / wr:.1f} per warp-row")
for r in hot:
    n = int(r["Instructions Executed"])
    print(r["Address"][-5:], f"{n / wr:5.2f}", r["Warp Stall Sampling (All Samples)"].rjust(5), r["Source"][:100])
