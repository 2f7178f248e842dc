"""Write profiles/<tag>_*.md from an ncu --set full report and a launch-list CSV
(ncu --metrics gpu__time_duration.sum), plus profiles/ncu_traffic.json entries."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def kernel_md(path, samples):
    hdr, units, data = raw(path)
    lines = []
    for r in data:
        d = dict(zip(hdr, r))
        lines.append(f"### `{d.get('Kernel Name')}`\n")
        lines.append("| metric | value |\n|---|---|")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k]} {units[hdr.index(k)]} |")
        rd = float(d["dram__bytes_read.sum"]); wr = float(d["dram__bytes_write.sum"])
        unit = units[hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
        traffic = (rd + wr) * scale
        inst = float(d["smsp__inst_executed.sum"])
        lines.append(f"| **traffic (read+write)** | {traffic / 1e6:.1f} MB |")
        lines.append(f"| warp instructions per channel-sample | {inst / samples:.3f} |")
        stalls = {k: float(d[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        lines.append("\nTop stall reasons (warps per issue-active cycle): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for k, v in top))
        lines.append("")
        return "\n".join(lines), traffic
    return "", None


def _inst(path):
    hdr, units, data = raw(path)
    return float(dict(zip(hdr, data[0]))["smsp__inst_executed.sum"])


def launches_md(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    order = []
    for r in data:
        if len(r) > iv:
            k = r[ik]
            if k not in agg:
                order.append(k)
            agg[k].append(float(r[iv].replace(",", "")) / 1e3)
    out = ["| kernel | launches | mean µs (cold, serialised) |", "|---|---|---|"]
    for k in order:
        v = agg[k]
        out.append(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v):.2f} |")
    step = [k for k in order if ("parse" in k or "decode" in k or "prep" in k) and len(agg[k]) >= 5]
    per = {k: sum(agg[k][-5:]) / len(agg[k][-5:]) for k in step}
    tot = sum(per.values())
    out.append("\nShare of one decode step (mean of the last launches of each step kernel): " + ", ".join(
        f"`{k.split('(')[0].replace('void ', '')}` {v:.1f} µs ({100 * v / tot:.1f}%)" for k, v in per.items()))
    return "\n".join(out)


if __name__ == "__main__":
    tag, gp = sys.argv[1], sys.argv[2]   # e.g. r1 gpurun_out/r1b
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    ij = os.path.join(ROOT, "profiles", "ncu_instr.json")
    instr = json.load(open(ij)) if os.path.exists(ij) else {}
    sys.path.insert(0, ROOT)
    import l3synth
    c2 = sum(3 * h * w for h, w in l3synth.imagenet_shapes(256))
    cases = {"c3_f32": ("c3_cityscapes_f32", 32 * 3 * 2048 * 1024, "C3 Cityscapes 32x2048x1024, fp32 out"),
             "c3_u8": ("c3_cityscapes_u8", 32 * 3 * 2048 * 1024, "C3 Cityscapes 32x2048x1024, u8 out"),
             "c4_u8": ("c4_uhd_u8", 16 * 3 * 3840 * 2160, "C4 UHD 16x3840x2160, u8 out (wide variant)"),
             "c2_u8": ("c2_imagenet_u8", c2, "C2 ImageNet-shaped 256 x ~500x375, u8 out"),
             "c3_f32_hwc": ("c3_cityscapes_f32_hwc", 32 * 3 * 2048 * 1024,
                            "C3 Cityscapes 32x2048x1024, fp32 HWC out (tile kernel, f3)")}
    for key, (tkey, samples, title) in cases.items():
        rep = f"{gp}_prof_{key}.ncu-rep"
        if not os.path.exists(rep):
            continue
        md, t = kernel_md(rep, samples)
        lines = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), rep, "30"],
                               capture_output=True, text=True).stdout
        traffic[tkey] = t
        instr[tkey] = \
            round(_inst(rep) / samples, 4)
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{key}.md"), "w") as f:
            f.write(f"# {tag}: ncu --set full, decode kernel, {title}\n\n")
            f.write(f"Source: `{os.path.basename(rep)}` (one launch, `-s 3 -c 1`, --clock-control none).\n\n")
            f.write(md)
            if lines:
                f.write("\n## Hottest source lines (share of warp instructions, share of stall samples)\n\n```\n")
                f.write(lines + "```\n")
    lc = f"{gp}_launches_c3_f32.csv"
    if os.path.exists(lc):
        with open(os.path.join(ROOT, "profiles", f"{tag}_launches_c3_f32.md"), "w") as f:
            f.write(f"# {tag}: launch list of `python bench.py --steps 5 --warmup 3` (C3 fp32) under\n"
                    "`ncu --metrics gpu__time_duration.sum --clock-control none`\n\n")
            f.write(launches_md(lc) + "\n")
    json.dump(traffic, open(tj, "w"), indent=1)
    instr["source"] = f"{tag}: smsp__inst_executed.sum / channel-samples of one launch (ncu --set full)"
    json.dump(instr, open(ij, "w"), indent=1)
    print(json.dumps(traffic))
