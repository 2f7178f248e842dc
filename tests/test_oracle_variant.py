"""Pins of the oracle's ablation format variant "L3IP" (original left/top/top-left Paeth,
SURVEY.md §8 f2, Fig. 10 `Baseline`; reading C16 in DESIGN.md).

The expected values come from hand derivations (tests/golden/png_paeth_variant.txt), an
algebraically rearranged form of the predictor swept over all 2^24 inputs, closed forms on
images whose residuals are known, and the independent bit-string model (oracle/pymodel.py).
"""
import struct

import numpy as np
import pytest

import l3synth
from conftest import hexbytes, read_golden
from oracle import l3ref, pymodel


def test_png_predictor_hand_examples():
    for v in read_golden("png_paeth_variant.txt")["predict"]:
        a, b, c, want = map(int, v.split())
        assert l3ref.predict_png(a, b, c) == want
        assert pymodel.predict_png(a, b, c) == want


def test_png_predictor_exhaustive_rearranged():
    """All 2^24 (a, b, c): since p-a = b-c, p-b = a-c, p-c = a+b-2c, the distances need no p."""
    idx = np.arange(1 << 24, dtype=np.int64)
    a, b, c = idx >> 16, (idx >> 8) & 255, idx & 255
    pa, pb, pc = np.abs(b - c), np.abs(a - c), np.abs(a + b - 2 * c)
    want = np.where((pa <= pb) & (pa <= pc), a, np.where(pb <= pc, b, c))
    got = l3ref.predict_png_many(a.astype(np.uint8), b.astype(np.uint8), c.astype(np.uint8))
    assert np.array_equal(got, want)


def test_worked_file_bytes():
    g = read_golden("png_paeth_variant.txt")
    img = np.broadcast_to(np.array([[10, 20], [30, 25]], np.uint8), (3, 2, 2)).copy()
    f = l3ref.encode_variant(img, N=2)
    assert f == hexbytes(g["file"])
    assert f[25:31] == hexbytes(g["patch_bytes"])
    assert pymodel.encode(img.tolist(), 2, predictor=1) == f
    st, dec = l3ref.decode_variant(f, (2, 2))
    assert st == l3ref.OK and np.array_equal(dec, img)


def test_vertical_constant_closed_form():
    """Every row equal to the previous one: the original Paeth predicts the top pixel exactly
    (p = b), so rows >= 1 are zero residual rows like a black image's: k = 1, base 0."""
    H, W, N = 40, 70, 32
    rng = np.random.default_rng(3)
    row = rng.integers(0, 256, (3, 1, W)).astype(np.uint8)
    img = np.repeat(row, H, axis=1)
    f = l3ref.encode_variant(img, N=N)
    gx, gy = -(-W // N), -(-H // N)
    total = 13 + 12 * gx * gy
    for ch in range(3):
        for p in range(gx * gy):
            x0, y0 = (p % gx) * N, (p // gx) * N
            w, h = min(N, W - x0), min(N, H - y0)
            seg = row[ch, 0, x0:x0 + w].astype(int)
            k0 = max(1, int(seg.max() - seg.min()).bit_length())
            total += -(-(12 + k0 * w + (h - 1) * (12 + w)) // 8)
    assert len(f) == total
    st, dec = l3ref.decode_variant(f, (H, W))
    assert st == l3ref.OK and np.array_equal(dec, img)


def test_horizontal_constant_closed_form():
    """Each row constant v_r: the original Paeth leaves only column 0 non-zero (v_r - v_{r-1}),
    where the custom Paeth gives that difference in every column."""
    H, W, N = 9, 16, 16
    v = np.array([0, 5, 9, 9, 2, 200, 201, 190, 60], np.uint8)
    img = np.broadcast_to(v[None, :, None], (3, H, W)).copy()
    f = l3ref.encode_variant(img, N=N)
    bits = 12 + 1 * W     # row 0: constant -> k = 1
    for r in range(1, H):
        d = (int(v[r]) - int(v[r - 1])) % 256
        s = d - 256 if d >= 128 else d
        lo, hi = min(0, s), max(0, s)
        bits += 12 + max(1, (hi - lo).bit_length()) * W
    assert len(f) == 13 + 12 + 3 * (-(-bits // 8))
    st, dec = l3ref.decode_variant(f, (H, W))
    assert st == l3ref.OK and np.array_equal(dec, img)


@pytest.mark.parametrize("seed", range(30))
def test_c_oracle_equals_pymodel_variant(seed):
    rng = np.random.default_rng(500 + seed)
    H, W = int(rng.integers(1, 14)), int(rng.integers(1, 14))
    N = int(rng.integers(1, 10))
    img = l3synth.uniform_image(H, W, seed) if seed % 2 else l3synth.natural(H, W, seed, 1.0)
    a = l3ref.encode_variant(img, N=N)
    assert a[:4] == b"L3IP"
    assert a == pymodel.encode(img.tolist(), N, predictor=1)
    assert np.array_equal(np.array(pymodel.decode(a), np.uint8), img)
    st, dec = l3ref.decode_variant(a, (H, W))
    assert st == l3ref.OK and np.array_equal(dec, img)


@pytest.mark.parametrize("shape,N", [((64, 64), 32), ((65, 129), 64), ((480, 640), 0), ((300, 257), 128)])
def test_variant_roundtrip_and_container(shape, N):
    H, W = shape
    img = l3synth.natural(H, W, 11, 1.0)
    f = l3ref.encode_variant(img, N=N)
    g = l3ref.encode(img, N=N)
    # same container: magic differs, W/H/N and the table length agree
    assert f[:4] == b"L3IP" and g[:4] == b"L3IF" and f[4:13] == g[4:13]
    st, dec = l3ref.decode_variant(f, shape)
    assert st == l3ref.OK and np.array_equal(dec, img)
    # the hot-path decoder's format is L3IF only: the strict oracle entry rejects L3IP
    assert l3ref.decode(f)[0] == l3ref.E_UNRECOGNIZED_FORMAT
    # and the variant entry also reads L3IF
    st, dec = l3ref.decode_variant(g, shape)
    assert st == l3ref.OK and np.array_equal(dec, img)


def test_variant_ratio_close_to_custom():
    """Both predictors exploit the same spatial redundancy: on natural-like content their
    compressed sizes agree within a few percent (PAPER.md:135 changes only the neighbours)."""
    img = l3synth.natural(1024, 2048, 2, l3synth.GAIN["cityscapes"])
    f, g = l3ref.encode_variant(img), l3ref.encode(img)
    assert 0.9 < len(f) / len(g) < 1.1
