"""Pins of the C oracle (oracle/l3ref.c) against what the paper and mathematics fix.

None of these re-types the oracle's own formula: each expected value comes from
the paper's printed numbers (tests/golden/*, cited), SPEC.md's worked vectors,
closed forms, an independently derived reformulation of the predictor, a second
pure-Python model built on bit strings, or exhaustive / brute-force sweeps.
"""
import struct

import numpy as np
import pytest

import l3synth
from conftest import hexbytes, read_golden
from oracle import l3ref, pymodel


# --------------------------------------------------------------------------- predictor

def test_fig3_worked_example():
    g = read_golden("fig3_paeth.txt")
    sel, orig, res = int(g["selected"]), int(g["original"]), int(g["residual"])
    # A previous row of [65, 65, 65] makes 65 the selected neighbour for the middle pixel.
    img = np.zeros((3, 2, 3), np.uint8)
    img[:, 0, :] = sel
    img[:, 1, :] = orig
    f = l3ref.encode(img, N=3)
    # row 1 residuals are all 74-65 = 9 -> k=1, base=9 (signed rule), deltas 0
    st, bad, dec, _ = l3ref.decode(f)
    assert st == l3ref.OK and (dec == img).all()
    k, base, deltas = l3ref.bd_encode_row(np.array([orig - sel] * 3), first_row=False)
    assert base == res and k == 1 and not deltas.any()
    assert (l3ref.predict(sel, sel, sel) + res) % 256 == orig


def test_spec_predictor_examples():
    for v in read_golden("fig3_paeth.txt")["predict"]:
        tl, t, tr, want = map(int, v.split())
        assert l3ref.predict(tl, t, tr) == want
        assert pymodel.predict(tl, t, tr) == want


def _reformulated(tl, t, tr):
    """Independent closed form (derived, not the paper's procedure):
    with a = TL-T and b = TR-T the distances are |b|, |a+b|, |a|. If T lies strictly
    between TL and TR (a*b < 0): TL when 2|b| <= |a|, TR when 2|a| < |b|, else T.
    Otherwise: TL when |b| <= |a|, else TR."""
    a = tl.astype(np.int32) - t
    b = tr.astype(np.int32) - t
    ua, ub = np.abs(a), np.abs(b)
    between = (a * b) < 0
    sel_between = np.where(2 * ub <= ua, tl, np.where(2 * ua < ub, tr, t))
    sel_outside = np.where(ub <= ua, tl, tr)
    return np.where(between, sel_between, sel_outside).astype(np.uint8)


def test_predictor_exhaustive_2_24():
    """All 2^24 (TL, T, TR) triples: oracle == independent reformulation."""
    idx = np.arange(1 << 24, dtype=np.uint32)
    tl = (idx >> 16).astype(np.uint8)
    t = ((idx >> 8) & 255).astype(np.uint8)
    tr = (idx & 255).astype(np.uint8)
    got = l3ref.predict_many(tl, t, tr)
    assert np.array_equal(got, _reformulated(tl, t, tr))


def test_predictor_properties():
    rng = np.random.default_rng(5)
    tl, t, tr = (rng.integers(0, 256, 200000).astype(np.uint8) for _ in range(3))
    p = l3ref.predict_many(tl, t, tr)
    assert np.all((p == tl) | (p == t) | (p == tr))          # membership
    # shift equivariance where the shifted triple stays in range
    c = rng.integers(-40, 41, len(t))
    ok = (np.minimum(np.minimum(tl, t), tr) + c >= 0) & (np.maximum(np.maximum(tl, t), tr) + c <= 255)
    s = l3ref.predict_many((tl + c)[ok], (t + c)[ok], (tr + c)[ok])
    assert np.array_equal(s.astype(int), p[ok].astype(int) + c[ok])


# --------------------------------------------------------------------------- base-delta

def test_bd_row_spec_example_and_bytes():
    g = read_golden("bd_row_spec_example.txt")
    row = np.array([int(x) for x in g["row"].split()], np.uint8)
    k, base, deltas = l3ref.bd_encode_row(row, first_row=True)
    assert (k, base) == (int(g["k"]), int(g["base"]))
    assert deltas.tolist() == [int(x) for x in g["deltas"].split()]
    img = np.broadcast_to(row, (3, 1, 4)).copy()
    f = l3ref.encode(img, N=4)
    assert f == hexbytes(g["file"])
    data = f[13 + 12:]
    assert data[:3] == hexbytes(g["patch_bytes"])
    bits = "".join(format(b, "08b") for b in data[:3])
    assert bits.startswith(g["bits"]) and set(bits[len(g["bits"]):]) <= {"0"}


def test_bd_row_spec_examples():
    assert l3ref.bd_encode_row(np.zeros(4), True)[:2] == (1, 0)
    k, b, d = l3ref.bd_encode_row(np.array([0, 255]), True)
    assert (k, b, d.tolist()) == (8, 0, [0, 255])
    # reading C2 (signed residual rows): [-1, 0, +1] -> base 0xFF, k = 2, deltas [0, 1, 2]
    k, b, d = l3ref.bd_encode_row(np.array([255, 0, 1]), False)
    assert (k, b, d.tolist()) == (2, 255, [0, 1, 2])
    # the same residual row under SPEC's unsigned reading spans 255 -> k = 8
    k, b, d = l3ref.bd_encode_row(np.array([255, 0, 1]), False, base_rule=l3ref.BASE_UNSIGNED)
    assert (k, b) == (8, 0)


def test_tiny_patch_sizes():
    g = read_golden("tiny_patches.txt")
    f = l3ref.encode(np.zeros((3, 2, 2), np.uint8), N=2)
    assert len(f) == 13 + 12 * 1 + 3 * 4
    assert f[25:29] == hexbytes(g["zero_2x2_patch_bytes"])
    f = l3ref.encode(np.full((3, 1, 1), 200, np.uint8), N=1)
    assert len(f) == 13 + 12 + 3 * 2
    assert f[25:27] == hexbytes(g["one_200_patch_bytes"])


# --------------------------------------------------------------------------- container

def test_policy_examples():
    assert l3ref.choose_patch_size(640, 480) == 32
    assert l3ref.choose_patch_size(3840, 2160) == 128
    assert l3ref.choose_patch_size(1920, 1080) == 128       # SPEC.md:188 (C10)
    assert l3ref.choose_patch_size(1280, 720) == 64
    assert l3ref.choose_patch_size(1079, 720) == 32
    assert l3ref.choose_patch_size(2048, 1024) == 128


@pytest.mark.parametrize("W,H,N,P", [(4, 4, 2, 4), (5, 3, 2, 6), (1920, 1080, 128, 135), (1, 1, 32, 1),
                                     (500, 375, 32, 192), (3840, 2160, 128, 510)])
def test_partition_and_header_length(W, H, N, P):
    img = np.zeros((3, H, W), np.uint8)
    f = l3ref.encode(img, N=N)
    st, _, _, (w, h, n, p) = l3ref.decode(f)
    assert st == l3ref.OK and (w, h, n, p) == (W, H, N, P)
    assert f[:4] == b"L3IF" and struct.unpack("<IIB", f[4:13]) == (W, H, N)
    offs = struct.unpack(f"<{3 * P}I", f[13:13 + 12 * P])
    assert offs[0] == 0 and all(a < b for a, b in zip(offs, offs[1:]))
    # all-zero patches: every row k=1 -> each patch ceil(h*(12+w)/8) bytes
    gx = -(-W // N)
    sizes = []
    for p in range(P):
        w = min(N, W - (p % gx) * N)
        h = min(N, H - (p // gx) * N)
        sizes.append(-(-(h * (12 + w)) // 8))
    assert len(f) == 13 + 12 * P + 3 * sum(sizes)


def test_black_fhd_closed_form():
    g = read_golden("table4_synthetic.txt")
    f = l3ref.encode(l3synth.black_image(1080, 1920))
    assert len(f) == int(g["black_fhd_file_bytes"])
    assert round(len(f) / (1920 * 1080 * 3), 2) in (0.13, 0.14)


def test_random_fhd_ratio_band():
    g = read_golden("table4_synthetic.txt")
    f = l3ref.encode(l3synth.random_image(1080, 1920, seed=0))
    r = len(f) / (1920 * 1080 * 3)
    assert float(g["random_fhd_ratio_lo"]) <= r <= float(g["random_fhd_ratio_hi"])


# --------------------------------------------------------------------------- second model / brute force

@pytest.mark.parametrize("seed", range(40))
def test_c_oracle_equals_pymodel_bytes(seed):
    rng = np.random.default_rng(100 + seed)
    H, W = int(rng.integers(1, 14)), int(rng.integers(1, 14))
    N = int(rng.integers(1, 10))
    img = l3synth.uniform_image(H, W, seed)
    signed = bool(seed % 2)
    rule = l3ref.BASE_SIGNED if signed else l3ref.BASE_UNSIGNED
    a = l3ref.encode(img, N=N, base_rule=rule)
    b = pymodel.encode(img.tolist(), N, signed_rule=signed)
    assert a == b
    assert np.array_equal(np.array(pymodel.decode(a), np.uint8), img)


def test_size_formula_against_pymodel_k():
    """file = 13 + 12P + sum ceil(sum_rows(12 + k*w)/8), k from the independent model."""
    for seed in range(20):
        img = l3synth.natural(37, 53, seed, 1.5)
        N = 16
        f = l3ref.encode(img, N=N)
        gx, gy = -(-53 // N), -(-37 // N)
        total = 13 + 12 * gx * gy
        for ch in range(3):
            for p in range(gx * gy):
                x0, y0 = (p % gx) * N, (p // gx) * N
                patch = [list(r[x0:x0 + N]) for r in img[ch, y0:y0 + N].tolist()]
                bits = sum(12 + pymodel.bd_row(rr, i == 0)[0] * len(rr)
                           for i, rr in enumerate(pymodel.filter_patch(patch)))
                total += -(-bits // 8)
        assert len(f) == total


def _roundtrip_columns(values, vertical):
    """Encode many single-channel tiny patches at once: N=2 strips."""
    n = len(values)
    per = -(-n // 3)
    vals = np.zeros((3 * per, values.shape[1]), np.uint8)
    vals[:n] = values
    vals = vals.reshape(3, per, values.shape[1])
    if vertical:   # patches of w=1, h=len: stack along H, W=1
        img = vals.reshape(3, per * values.shape[1], 1)
    else:          # patches of w=len, h=1: along W, H=1
        img = vals.reshape(3, 1, per * values.shape[1])
    f = l3ref.encode(img, N=values.shape[1])
    st, bad, dec, _ = l3ref.decode(f)
    assert st == l3ref.OK and np.array_equal(dec, img)
    return f


def test_exhaustive_tiny_patches():
    """All 1x1, 2x1 and 1x2 patches over all byte values roundtrip."""
    _roundtrip_columns(np.arange(256, dtype=np.uint8)[:, None], vertical=False)
    pairs = np.stack(np.meshgrid(np.arange(256), np.arange(256), indexing="ij"), -1).reshape(-1, 2).astype(np.uint8)
    f_h = _roundtrip_columns(pairs, vertical=False)
    f_v = _roundtrip_columns(pairs, vertical=True)
    # a vertical pair's second row is predicted from T only (reading C4): residual = b - a
    assert len(f_h) > 0 and len(f_v) > 0


@pytest.mark.parametrize("shape", [(1, 1), (3, 2), (17, 31), (64, 64), (65, 129), (480, 640)])
@pytest.mark.parametrize("N", [0, 1, 3, 32, 64, 128, 255])
def test_lossless_roundtrip(shape, N):
    H, W = shape
    if N in (1, 3) and H * W > 5000:
        pytest.skip("tiny N on large images is slow in the oracle")
    for seed in range(2):
        img = l3synth.uniform_image(H, W, seed * 7 + N)
        for rule, kx in ((l3ref.BASE_SIGNED, 0), (l3ref.BASE_UNSIGNED, 0), (l3ref.BASE_SIGNED, 2)):
            f = l3ref.encode(img, N=N, base_rule=rule, k_extra=kx)
            st, bad, dec, _ = l3ref.decode(f, exp_shape=(H, W))
            assert st == l3ref.OK and bad == -1 and np.array_equal(dec, img)


def test_ratio_reading_c2_natural_content():
    """Reading C2: the signed base lands natural content inside Table 4's range (0.33-0.76,
    PAPER.md:259) while the unsigned reading leaves it ~incompressible."""
    img = l3synth.make_batch("c3_cityscapes", 1)[0]
    rs = len(l3ref.encode(img)) / img.size
    ru = len(l3ref.encode(img, base_rule=l3ref.BASE_UNSIGNED)) / img.size
    assert 0.40 <= rs <= 0.48
    assert ru > 0.9


# --------------------------------------------------------------------------- errors

def _file(seed=0, H=40, W=70, N=16):
    img = l3synth.natural(H, W, seed, 2.0)
    return img, bytearray(l3ref.encode(img, N=N))


def test_error_taxonomy():
    img, f = _file()
    P = 3 * 5
    assert l3ref.decode(bytes(f))[0] == l3ref.OK
    bad = bytearray(f); bad[0:4] = b"PNG\x00"
    assert l3ref.decode(bytes(bad))[0] == l3ref.E_UNRECOGNIZED_FORMAT
    assert l3ref.decode(b"L3")[0] == l3ref.E_UNRECOGNIZED_FORMAT
    assert l3ref.decode(bytes(f[:10]))[0] == l3ref.E_CORRUPT_HEADER
    assert l3ref.decode(bytes(f[:13 + 12 * P - 1]))[0] == l3ref.E_CORRUPT_HEADER
    assert l3ref.decode(bytes(f), exp_shape=(40, 71))[0] == l3ref.E_CORRUPT_HEADER
    # non-monotonic offsets
    offs = list(struct.unpack(f"<{3 * P}I", f[13:13 + 12 * P]))
    o2 = offs[:]; o2[5], o2[6] = o2[6], o2[5]
    bad = bytearray(f); bad[13:13 + 12 * P] = struct.pack(f"<{3 * P}I", *o2)
    assert l3ref.decode(bytes(bad))[0] == l3ref.E_CORRUPT_HEADER
    # k = 0 in unit 7's first row -> CORRUPT_STREAM at unit 7
    data0 = 13 + 12 * P
    bad = bytearray(f); bad[data0 + offs[7]] &= 0x0F
    st, u, _, _ = l3ref.decode(bytes(bad))
    assert (st, u) == (l3ref.E_CORRUPT_STREAM, 7)
    # k = 9 in unit 20 and k = 0 in unit 30: the first unit wins
    bad = bytearray(f)
    bad[data0 + offs[20]] = (bad[data0 + offs[20]] & 0x0F) | 0x90
    bad[data0 + offs[30]] &= 0x0F
    st, u, _, _ = l3ref.decode(bytes(bad))
    assert (st, u) == (l3ref.E_CORRUPT_STREAM, 20)
    # truncating the file cuts the last unit's stream
    st, u, _, _ = l3ref.decode(bytes(f[:-3]))
    assert (st, u) == (l3ref.E_TRUNCATED_STREAM, 3 * P - 1)


def test_batch_threads_and_order():
    imgs = [l3synth.uniform_image(h, w, s) for s, (h, w) in enumerate([(30, 50), (1, 1), (64, 64), (33, 7)])]
    files = [l3ref.encode(im, N=16) for im in imgs]
    files[2] = b"XXXX" + files[2][4:]
    src = np.frombuffer(b"".join(files), np.uint8)
    offs = np.cumsum([0] + [len(f) for f in files]).astype(np.uint64)
    shapes = np.array([im.shape[1:] for im in imgs], np.int32)
    r1 = l3ref.decode_batch(src, offs, shapes, threads=1)
    r4 = l3ref.decode_batch(src, offs, shapes, threads=4)
    assert r1[1].tolist() == r4[1].tolist() == [0, 0, l3ref.E_UNRECOGNIZED_FORMAT, 0]
    for i in (0, 1, 3):
        assert np.array_equal(r1[0][i], imgs[i]) and np.array_equal(r4[0][i], imgs[i])


# --------------------------------------------------------------------------- normalisation (reading C14)

def test_normalize_closed_form():
    mean, std = [0.485, 0.456, 0.406], [0.229, 0.224, 0.225]
    x = np.zeros((3, 1, 2), np.uint8); x[:, 0, 1] = 255
    y = l3ref.normalize(x, mean, std)
    for c in range(3):
        assert y[c, 0, 0] == pytest.approx(-mean[c] / std[c], abs=1e-15)
        assert y[c, 0, 1] == pytest.approx((1 - mean[c]) / std[c], abs=1e-15)
