"""Per-source-line instruction counts and stall samples from an ncu report (needs -lineinfo and
--import-source on): python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[2:], rec[2:]))
    try:
        inst = int(d.get("Instructions Executed", "0") or 0)
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    rows.append((inst, samp, fname, rec[0], rec[1].strip()[:90]))
tot_i = sum(r[0] for r in rows) or 1
tot_s = sum(r[1] for r in rows) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for inst, samp, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * inst / tot_i:5.1f}% {100 * samp / tot_s:5.1f}%  {f}:{ln}  {src}")
