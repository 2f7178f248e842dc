"""Instruction mix of the row loops of the decode kernels (static SASS, no GPU needed).

usage: python scripts/sass_loops.py [LIB.so] [kernel-substring]

Finds every backward branch whose body holds a VIMNMX3 (the predictor's 3-way
minimum, i.e. a row loop), and prints its length and opcode mix. The row loops
unroll two rows, so the instructions per row are half the body length; per
sample, a quarter of that (4 columns per lane).
"""
from __future__ import annotations

import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def functions(lib: str) -> dict[str, list[tuple[int, str]]]:
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    out: dict[str, list[tuple[int, str]]] = {}
    cur = None
    for line in sass.split("\n"):
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", line)
        if m and cur:
            out[cur].append((int(m.group(1), 16), m.group(2).strip()))
    return out


def row_loops(ins: list[tuple[int, str]]):
    addr = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA.*?(0x[0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr:
            body = ins[addr[tgt]:i + 1]
            if any(("VIMNMX3" in x or "HMUL2" in x or "HMNMX2" in x) for _, x in body) and len(body) < 800:
                yield tgt, a, body


def main() -> None:
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2208_08711_b200", "libl3_b200.so")
    pat = sys.argv[2] if len(sys.argv) > 2 else "l3_decode_kernel"
    for name, ins in functions(lib).items():
        if pat not in name:
            continue
        print(name)
        for tgt, a, body in row_loops(ins):
            ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0] for _, x in body)
            print(f"  loop {tgt:#x}-{a:#x}: {len(body)} instr, VIMNMX3 x{ops['VIMNMX3.U16x2']}, "
                  f"HMUL2 x{ops['HMUL2']}, LDL/STL {ops['LDL'] + ops['STL']}")
            print("    " + ", ".join(f"{k} {v}" for k, v in ops.most_common(14)))


if __name__ == "__main__":
    main()


# Pipe classes (sm_100a, approximate): the half-rate ALU pipe vs the FMA-heavy pipe (IMAD).
ALU = ("LOP3", "PRMT", "SHF", "VABSDIFF4", "VIMNMX", "ISETP", "SEL", "IADD3", "LEA", "VIADDMNMX", "FLO", "POPC",
       "PLOP3", "BMSK", "IABS")
FMA = ("IMAD", "FFMA", "FMUL", "FADD")


def pipe_mix(body) -> dict[str, int]:
    mix = collections.Counter()
    for _, x in body:
        op = re.sub(r"^@!?U?P\w+\s+", "", x).split()[0]
        base = op.split(".")[0]
        if op.startswith("VIADDMNMX"):
            mix["alu"] += 1
        elif base in ALU:
            mix["alu"] += 1
        elif base in FMA:
            mix["fma"] += 1
        elif base == "VIADD":
            mix["viadd"] += 1
        else:
            mix["other"] += 1
    return dict(mix)


def mix_report(lib: str, pat: str) -> None:
    """ALU / FMA-class / other op counts of each row loop (python -c 'import scripts.sass_loops as s; ...')."""
    half = ("HADD2", "HFMA2", "HMUL2", "HMNMX2")
    for name, ins in functions(lib).items():
        if pat not in name:
            continue
        for tgt, a, body in row_loops(ins):
            c = collections.Counter()
            for _, x in body:
                op = re.sub(r"^@!?U?P\w+\s+", "", x).split()[0]
                b = op.split(".")[0]
                if b in ALU or op.startswith("VIMNMX") or op.startswith("VIADD"):
                    c["alu"] += 1
                elif b in FMA:
                    c["fma"] += 1
                elif b in half:
                    c["half"] += 1
                else:
                    c["other"] += 1
            print(f"{name[:60]} {tgt:#x}: {len(body)} instr {dict(c)}")
