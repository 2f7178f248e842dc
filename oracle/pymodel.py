"""Second, independent pure-Python model of the L3 codec — TINY INPUTS ONLY.

TEST INFRASTRUCTURE ONLY. It exists to pin the C oracle (oracle/l3ref.c) on
brute-force cases: it keeps the bitstream as a Python string of '0'/'1'
characters (so MSB-first order is visible by eye) and uses the predictor's
*definition* as a sort over (distance, tie rank) instead of the C loop.
Citations: PAPER.md:135-139 (§4.2 Fig. 3), :150-152 (§4.2 Fig. 4),
:166-168 (§4.3 Fig. 5). Readings C1..C14: DESIGN.md §3.
"""
from __future__ import annotations

import struct


def predict(tl: int, t: int, tr: int) -> int:
    """closest of (TL, T, TR) to TL+TR-T; ties in that order (C3)."""
    ref = tl + tr - t
    ranked = sorted([(abs(tl - ref), 0, tl), (abs(t - ref), 1, t), (abs(tr - ref), 2, tr)])
    return ranked[0][2]


def predict_png(a: int, b: int, c: int) -> int:
    """PNG Paeth (original L3 ablation baseline): closest to a+b-c, ties a, b, c."""
    p = a + b - c
    return sorted([(abs(p - a), 0, a), (abs(p - b), 1, b), (abs(p - c), 2, c)])[0][2]


def filter_patch_png(patch):
    """Original-Paeth residuals of a patch: row 0 raw; left / top-left are 0 at column 0 (reading C16)."""
    out = [list(patch[0])]
    for r in range(1, len(patch)):
        row = []
        for c in range(len(patch[r])):
            a = patch[r][c - 1] if c else 0
            cc = patch[r - 1][c - 1] if c else 0
            row.append((patch[r][c] - predict_png(a, patch[r - 1][c], cc)) % 256)
        out.append(row)
    return out


def _neighbours(prev, c):
    w = len(prev)
    t = prev[c]
    tl = prev[c - 1] if c > 0 else t           # C4: clamp to edge
    tr = prev[c + 1] if c < w - 1 else t
    return tl, t, tr


def filter_patch(patch):
    """patch: list of rows (lists of ints). Returns residual rows (C1, C5)."""
    out = [list(patch[0])]
    for r in range(1, len(patch)):
        out.append([(patch[r][c] - predict(*_neighbours(patch[r - 1], c))) % 256
                    for c in range(len(patch[r]))])
    return out


def bd_row(res, first_row: bool, signed_rule: bool = True):
    """base = minimum, k = bits covering the deltas (C2, C6)."""
    vals = [v - 256 if (signed_rule and not first_row and v >= 128) else v for v in res]
    mn, mx = min(vals), max(vals)
    k = max(1, (mx - mn).bit_length())
    base = mn % 256
    return k, base, [(v - base) % 256 for v in res]


def encode(planar, N: int, signed_rule: bool = True, predictor: int = 0) -> bytes:
    """planar: [3][H][W] nested lists. Returns L3 file bytes (C8, C9).
    predictor 1 = original Paeth ablation variant, magic "L3IP" (reading C16)."""
    H, W = len(planar[0]), len(planar[0][0])
    gx, gy = -(-W // N), -(-H // N)
    P = gx * gy
    bits_per_unit = []
    for ch in range(3):
        for p in range(P):
            x0, y0 = (p % gx) * N, (p // gx) * N
            patch = [row[x0:x0 + N] for row in planar[ch][y0:y0 + N]]
            bits = ""
            for r, rres in enumerate(filter_patch_png(patch) if predictor else filter_patch(patch)):
                k, base, deltas = bd_row(rres, r == 0, signed_rule)
                bits += format(k, "04b") + format(base, "08b") + "".join(format(d, f"0{k}b") for d in deltas)
            bits += "0" * (-len(bits) % 8)                # byte-align each patch
            bits_per_unit.append(bits)
    offsets, data, pos = [], b"", 0
    for bits in bits_per_unit:
        offsets.append(pos)
        chunk = bytes(int(bits[i:i + 8], 2) for i in range(0, len(bits), 8))
        data += chunk
        pos += len(chunk)
    magic = b"L3IP" if predictor else b"L3IF"
    return magic + struct.pack("<IIB", W, H, N) + struct.pack(f"<{3 * P}I", *offsets) + data


def decode(blob: bytes):
    """Returns [3][H][W] nested lists (valid files only)."""
    assert blob[:4] in (b"L3IF", b"L3IP")
    png = blob[:4] == b"L3IP"
    W, H, N = struct.unpack("<IIB", blob[4:13])
    gx, gy = -(-W // N), -(-H // N)
    P = gx * gy
    offs = list(struct.unpack(f"<{3 * P}I", blob[13:13 + 12 * P]))
    data = blob[13 + 12 * P:]
    out = [[[0] * W for _ in range(H)] for _ in range(3)]
    for u in range(3 * P):
        ch, p = divmod(u, P)
        seg = data[offs[u]:(offs[u + 1] if u + 1 < 3 * P else len(data))]
        bits = "".join(format(b, "08b") for b in seg)
        x0, y0 = (p % gx) * N, (p // gx) * N
        w, h = min(N, W - x0), min(N, H - y0)
        pos = 0
        prev = None
        for r in range(h):
            k = int(bits[pos:pos + 4], 2)
            base = int(bits[pos + 4:pos + 12], 2)
            pos += 12
            res = []
            for _ in range(w):
                res.append((base + int(bits[pos:pos + k], 2)) % 256)
                pos += k
            if prev is None:
                row = res
            elif png:
                row = []
                for c in range(w):
                    a = row[c - 1] if c else 0
                    cc = prev[c - 1] if c else 0
                    row.append((predict_png(a, prev[c], cc) + res[c]) % 256)
            else:
                row = [(predict(*_neighbours(prev, c)) + res[c]) % 256 for c in range(w)]
            out[ch][y0 + r][x0:x0 + w] = row
            prev = row
    return out
