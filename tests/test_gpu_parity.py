"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

u8 output must be bit-exact; fused fp32 output within 1e-6 absolute of the oracle's
fp64 normalisation (BASELINE.json north_star); status / bad_unit identical to the
oracle's sequential decode on corrupted input.
"""
import numpy as np
import pytest
import torch

import l3synth
from oracle import l3ref

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2208_08711_b200 import BatchDecoder, encode_batch, normalize_constants, pack_files  # noqa: E402
from paper_2208_08711_b200.api import IMAGENET_MEAN, IMAGENET_STD  # noqa: E402

F32_TOL = 1e-6


def gpu_decode(files, shapes, dtype=torch.uint8, scale=(1, 1, 1), bias=(0, 0, 0), canary=True, gap=0, wide=False,
               layout="chw"):
    """Decode files on the GPU into per-image blocks (optionally separated by `gap` canary
    elements). Returns (list of arrays [3,H,W], status, bad_unit, flat output)."""
    src, offs = pack_files(files)
    n = len(files)
    sizes = [3 * h * w for h, w in shapes]
    out_off = np.zeros(n, np.int64)
    for i in range(1, n):
        out_off[i] = out_off[i - 1] + sizes[i - 1] + gap
    total = int(out_off[-1] + sizes[-1] + gap) if n else 1
    fill = 0xA5 if dtype == torch.uint8 else float("nan")
    out = torch.full((total,), fill, dtype=dtype, device="cuda")
    dec = BatchDecoder(max(n, 1))
    sh = torch.tensor(np.array(shapes, np.int32).reshape(n, 2), device="cuda")
    st, bad = dec.decode(src, offs, sh, out, out_offsets=torch.from_numpy(out_off).cuda(), scale=scale, bias=bias,
                         wide=wide, layout=layout)
    torch.cuda.synchronize()
    flat = out.cpu().numpy()
    imgs = [flat[int(o):int(o) + s].reshape(3, h, w) for o, s, (h, w) in zip(out_off, sizes, shapes)]
    return imgs, st.cpu().numpy(), bad.cpu().numpy(), flat, out_off, sizes


def check_u8(imgs_ref, files, gap=7):
    """u8 parity through both u8 kernel variants (narrow and L3_DECODE_HINT_WIDE)."""
    for wide in (False, True):
        _check_u8(imgs_ref, files, gap, wide)


def _check_u8(imgs_ref, files, gap, wide):
    shapes = [im.shape[1:] for im in imgs_ref]
    got, st, bad, flat, out_off, sizes = gpu_decode(files, shapes, gap=gap, wide=wide)
    assert st.tolist() == [0] * len(files), st
    for i, (g, r) in enumerate(zip(got, imgs_ref)):
        if not np.array_equal(g, r):
            diff = np.argwhere(g != r)
            raise AssertionError(f"image {i} shape {r.shape}: {len(diff)} mismatches, first {diff[:5].tolist()}")
    # canary: gaps between images untouched -> every output byte written exactly where expected
    mask = np.ones(flat.shape, bool)
    for o, s in zip(out_off, sizes):
        mask[int(o):int(o) + s] = False
    assert (flat[mask] == 0xA5).all()


# ------------------------------------------------------------------ configs

def test_config1_64x64_gradient():
    im = l3synth.make_batch("c1_64x64")[0]
    f = l3ref.encode(im)
    st, _, ref, _ = l3ref.decode(f)
    assert st == 0
    check_u8([ref], [f])


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (7, 1), (2, 2), (17, 31), (31, 17), (65, 129), (129, 65),
                                   (33, 250), (300, 257)])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8, 16, 31, 32, 33, 64, 100, 127, 128, 129, 200, 255])
def test_shapes_and_patch_sizes(shape, N):
    H, W = shape
    if N <= 3 and H * W > 4000:
        pytest.skip("tiny N on large images: covered by smaller shapes")
    imgs, files = [], []
    for s in range(2):
        im = l3synth.uniform_image(H, W, seed=1000 * N + s)
        rule = l3ref.BASE_SIGNED if s == 0 else l3ref.BASE_UNSIGNED
        files.append(l3ref.encode(im, N=N, base_rule=rule, k_extra=s))
        st, _, ref, _ = l3ref.decode(files[-1])
        assert st == 0
        imgs.append(ref)
    check_u8(imgs, files)


def test_mixed_batch_many_shapes():
    rng = np.random.default_rng(3)
    imgs, files = [], []
    for i in range(60):
        H, W = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        N = int(rng.choice([0, 1, 7, 16, 32, 64, 128, 150, 255])) if H * W < 20000 else int(rng.choice([0, 32, 128]))
        im = l3synth.uniform_image(H, W, seed=i)
        files.append(l3ref.encode(im, N=N, k_extra=int(rng.integers(0, 3)) if i % 3 == 0 else 0))
        imgs.append(im)
    check_u8(imgs, files)


def test_extremes_black_random():
    imgs = [l3synth.black_image(1080, 1920), l3synth.random_image(1080, 1920, 0), l3synth.black_image(3, 5)]
    check_u8(imgs, [l3ref.encode(im) for im in imgs])


def test_config2_imagenet_batch():
    imgs = l3synth.make_batch("c2_imagenet")
    check_u8(imgs, [l3ref.encode(im) for im in imgs], gap=0)


def test_config3_cityscapes_full_fp32_and_u8():
    """Full config 3 batch (32 x 2048x1024), dense [n,3,H,W] output as bench.py runs it."""
    imgs = l3synth.make_batch("c3_cityscapes")
    files = [l3ref.encode(im) for im in imgs]
    src, offs = pack_files(files)
    n = len(imgs)
    dec = BatchDecoder(n)
    sh = torch.tensor([[1024, 2048]] * n, dtype=torch.int32, device="cuda")
    out = torch.empty((n, 3, 1024, 2048), dtype=torch.uint8, device="cuda")
    refs = []
    for i in range(n):
        st_o, _, ref, _ = l3ref.decode(files[i])
        assert st_o == 0
        refs.append(ref)
    for wide in (False, True):
        out.fill_(0xA5)
        st, _ = dec.decode(src, offs, sh, out, wide=wide)
        torch.cuda.synchronize()
        assert st.cpu().tolist() == [0] * n
        got = out.cpu().numpy()
        for i in range(n):
            assert np.array_equal(got[i], refs[i]), (wide, i)
    scale, bias = normalize_constants(IMAGENET_MEAN, IMAGENET_STD)
    outf = torch.empty((n, 3, 1024, 2048), dtype=torch.float32, device="cuda")
    st, _ = dec.decode(src, offs, sh, outf, scale=scale, bias=bias)
    torch.cuda.synchronize()
    assert st.cpu().tolist() == [0] * n
    # every image's sampled rows checked against the oracle's fp64 normalisation
    rng = np.random.default_rng(0)
    gf = outf.cpu().numpy()
    for i in range(n):
        rows = rng.integers(0, 1024, 16)
        ref = l3ref.normalize(imgs[i][:, rows, :], IMAGENET_MEAN, IMAGENET_STD)
        assert np.abs(gf[i][:, rows, :].astype(np.float64) - ref).max() <= F32_TOL
    ref0 = l3ref.normalize(imgs[0], IMAGENET_MEAN, IMAGENET_STD)
    assert np.abs(gf[0].astype(np.float64) - ref0).max() <= F32_TOL


def test_config4_uhd_full_batch():
    """The whole config-4 batch (16 x 3840x2160, the bench's workload) through both u8 kernel variants
    (the bench times the wide one), bit-exact against the oracle's encode -> the GPU decode."""
    imgs = l3synth.make_batch("c4_uhd")
    assert len(imgs) == 16
    check_u8(imgs, [l3ref.encode(im) for im in imgs], gap=0)


def test_fp32_all_values_and_ragged():
    """All 256 byte values in every channel, odd widths (scalar-store path)."""
    base = np.arange(256, dtype=np.uint8)
    im = np.stack([np.tile(base, (3, 1)) for _ in range(3)])[:, :, :253]
    im2 = l3synth.uniform_image(77, 333, 5)
    files = [l3ref.encode(im, N=16), l3ref.encode(im2)]
    scale, bias = normalize_constants(IMAGENET_MEAN, IMAGENET_STD)
    got, st, _, _, _, _ = gpu_decode(files, [im.shape[1:], im2.shape[1:]], torch.float32, scale, bias, gap=3)
    assert st.tolist() == [0, 0]
    for g, r in zip(got, [im, im2]):
        ref = l3ref.normalize(r, IMAGENET_MEAN, IMAGENET_STD)
        assert np.abs(g.astype(np.float64) - ref).max() <= F32_TOL


# ------------------------------------------------------------------ faults (a7)

def _corrupt_variants(rng, f, P):
    data0 = 13 + 12 * 3 * P // 3
    out = []
    b = bytearray(f); b[0] ^= 0xFF; out.append(bytes(b))                     # magic
    out.append(bytes(f[:10]))                                                # short header
    out.append(bytes(f[:data0 - 1]))                                         # truncated offsets
    out.append(bytes(f[:-int(rng.integers(1, 40))]))                         # truncated stream
    b = bytearray(f); b[13 + 4 * 3:13 + 4 * 4] = b[13:17]; out.append(bytes(b))   # non-monotonic offsets
    for _ in range(6):                                                       # random byte flips in data
        b = bytearray(f)
        for _ in range(int(rng.integers(1, 4))):
            j = int(rng.integers(data0, len(b)))
            b[j] = int(rng.integers(0, 256))
        out.append(bytes(b))
    b = bytearray(f)                                                         # k = 0 at a unit start
    offs = np.frombuffer(bytes(f[13:data0]), "<u4")
    u = int(rng.integers(0, len(offs)))
    b[data0 + int(offs[u])] &= 0x0F
    out.append(bytes(b))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_fault_injection_status_parity(seed):
    rng = np.random.default_rng(seed)
    H, W = int(rng.integers(20, 200)), int(rng.integers(20, 300))
    N = int(rng.choice([8, 16, 32, 64, 128, 200]))
    im = l3synth.natural(H, W, seed, 3.0)
    f = l3ref.encode(im, N=N)
    P = (-(-W // N)) * (-(-H // N))
    files = _corrupt_variants(rng, f, P) + [f]
    shapes = [(H, W)] * len(files)
    for dtype, wide, layout in ((torch.uint8, False, "chw"), (torch.uint8, True, "chw"), (torch.float32, False, "chw"),
                                (torch.uint8, False, "hwc"), (torch.float32, False, "hwc")):
        _, st, bad, _, _, _ = gpu_decode(files, shapes, dtype=dtype, wide=wide, layout=layout)
        for i, fi in enumerate(files):
            rst, rbad, _, _ = l3ref.decode(fi, exp_shape=(H, W))
            assert (st[i], bad[i]) == (rst, rbad), (dtype, wide, layout, i, st[i], bad[i], rst, rbad)


@pytest.mark.parametrize("seed", range(3))
def test_a1_launch_modes_agree(seed):
    """The same corrupted batch through both a1 modes: inside every decode CTA (n <= 32, one launch) and
    the a1 kernel + PDL (the batch repeated to n > 32): statuses, bad units and pixels equal the oracle's."""
    from paper_2208_08711_b200 import l3
    rng = np.random.default_rng(100 + seed)
    H, W = int(rng.integers(20, 200)), int(rng.integers(20, 300))
    files, shapes = [], []
    for N in (32, 64, 128, 200):   # every decode mode incl. the generic N > 128 path
        im = l3synth.natural(H, W, seed + N, 3.0)
        f = l3ref.encode(im, N=N)
        P = (-(-W // N)) * (-(-H // N))
        v = _corrupt_variants(rng, f, P)
        files += [v[0], v[3], v[4], v[5], v[-1], f]   # header, truncation, offsets, data flips, k = 0, valid
    shapes = [(H, W)] * len(files)
    assert len(files) <= 32
    big = files * (-(-40 // len(files)))   # > 32 images: the a1 kernel path
    for dtype, wide in ((torch.uint8, False), (torch.uint8, True), (torch.float32, False)):
        for fs in (files, big):
            out, st, bad, _, _, _ = gpu_decode(fs, [(H, W)] * len(fs), dtype=dtype, wide=wide)
            for i, fi in enumerate(fs):
                rst, rbad, rpix, _ = l3ref.decode(fi, exp_shape=(H, W))
                assert (st[i], bad[i]) == (rst, rbad), (dtype, wide, len(fs), i, st[i], bad[i], rst, rbad)
                if rst == 0 and dtype == torch.uint8:
                    assert np.array_equal(out[i], np.asarray(rpix).reshape(3, H, W)), (wide, len(fs), i)
    # the launch count that l3_decode_launches reports for the two modes
    dec = BatchDecoder(len(big))
    src, offs = pack_files(big)
    sh = torch.tensor(np.array([(H, W)] * len(big), np.int32), device="cuda")
    o = torch.empty(len(big) * 3 * H * W, dtype=torch.uint8, device="cuda")
    assert l3.l3_decode_launches(dec.args(src, offs, sh, o)) == 2
    src, offs = pack_files(files)
    assert l3.l3_decode_launches(dec.args(src, offs, sh[:len(files)].contiguous(), o)) == 1


def test_shape_mismatch_is_corrupt_header():
    im = l3synth.natural(40, 50, 1, 1.0)
    f = l3ref.encode(im)
    _, st, bad, _, _, _ = gpu_decode([f, f], [(40, 50), (40, 51)])
    assert st.tolist() == [0, 3] and bad.tolist() == [-1, -1]


# ------------------------------------------------------------------ GPU encoder (f4)

@pytest.mark.parametrize("seed", range(4))
def test_gpu_encoder_byte_identical(seed):
    rng = np.random.default_rng(seed)
    imgs, Ns = [], []
    for i in range(12):
        H, W = int(rng.integers(1, 260)), int(rng.integers(1, 260))
        imgs.append(l3synth.uniform_image(H, W, 100 * seed + i))
        Ns.append(int(rng.choice([0, 1, 5, 16, 32, 64, 128, 200, 255])) if H * W < 30000 else 0)
    src, offs = encode_batch(imgs, patch_sizes=Ns)
    torch.cuda.synchronize()
    o = offs.cpu().numpy()
    buf = src.cpu().numpy()
    for i, (im, N) in enumerate(zip(imgs, Ns)):
        want = l3ref.encode(im, N=N)
        got = buf[o[i]:o[i + 1]].tobytes()
        assert got == want, (i, im.shape, N, len(got), len(want))


def test_gpu_encoder_config3_identical():
    imgs = l3synth.make_batch("c3_cityscapes", 4)
    src, offs = encode_batch(imgs)
    o = offs.cpu().numpy()
    buf = src.cpu().numpy()
    for i, im in enumerate(imgs):
        assert buf[o[i]:o[i + 1]].tobytes() == l3ref.encode(im)


def test_device_predictor_exhaustive_2_24():
    """The kernel's pair-form (SWAR) predictor equals the oracle on all 2^24 triples."""
    from paper_2208_08711_b200 import l3
    out = torch.empty(1 << 24, dtype=torch.uint8, device="cuda")
    l3.l3_selftest_paeth(out)
    torch.cuda.synchronize()
    idx = np.arange(1 << 24, dtype=np.uint32)
    ref = l3ref.predict_many((idx >> 16).astype(np.uint8), ((idx >> 8) & 255).astype(np.uint8),
                             (idx & 255).astype(np.uint8))
    got = out.cpu().numpy()
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, [(int(i) >> 16, (int(i) >> 8) & 255, int(i) & 255, int(got[i]), int(ref[i])) for i in bad[:8]]


def test_device_predictor_h2_exhaustive_2_24():
    """The kernel's biased-half (fp16x2) predictor equals the oracle on all 2^24 triples."""
    from paper_2208_08711_b200 import l3
    out = torch.empty(1 << 24, dtype=torch.uint8, device="cuda")
    l3.l3_selftest_paeth_h2(out)
    torch.cuda.synchronize()
    idx = np.arange(1 << 24, dtype=np.uint32)
    ref = l3ref.predict_many((idx >> 16).astype(np.uint8), ((idx >> 8) & 255).astype(np.uint8),
                             (idx & 255).astype(np.uint8))
    got = out.cpu().numpy()
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, [(int(i) >> 16, (int(i) >> 8) & 255, int(i) & 255, int(got[i]), int(ref[i])) for i in bad[:8]]


def test_device_predictor4_exhaustive_2_24():
    """The kernel's byte-form 4-sample predictor equals the oracle on all 2^24 triples,
    at each of the 4 sample positions of a lane (neighbouring columns hashed)."""
    from paper_2208_08711_b200 import l3
    out = torch.empty(4 << 24, dtype=torch.uint8, device="cuda")
    l3.l3_selftest_paeth4(out)
    torch.cuda.synchronize()
    idx = np.arange(1 << 24, dtype=np.uint32)
    ref = l3ref.predict_many((idx >> 16).astype(np.uint8), ((idx >> 8) & 255).astype(np.uint8),
                             (idx & 255).astype(np.uint8))
    got = out.cpu().numpy().reshape(4, 1 << 24)
    for q in range(4):
        bad = np.flatnonzero(got[q] != ref)
        assert bad.size == 0, (q, [(int(i) >> 16, (int(i) >> 8) & 255, int(i) & 255, int(got[q][i]), int(ref[i]))
                                   for i in bad[:8]])


# ------------------------------------------------------------------ f3: partial decode (crop / flip)

def _crop_decode(files, shapes, crops, dtype=torch.uint8, scale=(1, 1, 1), bias=(0, 0, 0), layout="chw",
                 use_crops=True):
    """Decode into per-image window blocks; returns planar [3, h, w] arrays whatever the layout."""
    src, offs = pack_files(files)
    n = len(files)
    sizes = [3 * int(c[2]) * int(c[3]) for c in crops]
    oo = np.zeros(n, np.int64)
    oo[1:] = np.cumsum(sizes)[:-1]
    fill = 0xA5 if dtype == torch.uint8 else float("nan")
    out = torch.full((sum(sizes),), fill, dtype=dtype, device="cuda")
    dec = BatchDecoder(n)
    sh = torch.tensor(np.array(shapes, np.int32).reshape(n, 2), device="cuda")
    cr = torch.tensor(np.array(crops, np.int32).reshape(n, 5), device="cuda") if use_crops else None
    st, bad = dec.decode(src, offs, sh, out, out_offsets=torch.from_numpy(oo).cuda(), scale=scale, bias=bias,
                         crops=cr, layout=layout)
    torch.cuda.synchronize()
    flat = out.cpu().numpy()
    if layout == "hwc":
        blocks = [flat[int(o):int(o) + s].reshape(int(c[2]), int(c[3]), 3).transpose(2, 0, 1)
                  for o, s, c in zip(oo, sizes, crops)]
    else:
        blocks = [flat[int(o):int(o) + s].reshape(3, int(c[2]), int(c[3])) for o, s, c in zip(oo, sizes, crops)]
    return blocks, st.cpu().numpy()


def _window(img, c):
    y, x, h, w, flip = c
    v = img[:, y:y + h, x:x + w]
    return v[:, :, ::-1] if flip else v


@pytest.mark.parametrize("seed", range(4))
def test_crop_flip_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    imgs, files, crops = [], [], []
    for i in range(10):
        H, W = int(rng.integers(1, 400)), int(rng.integers(1, 400))
        N = int(rng.choice([0, 5, 16, 32, 64, 100, 128, 160, 255]))
        im = l3synth.uniform_image(H, W, 50 * seed + i)
        imgs.append(im)
        files.append(l3ref.encode(im, N=N))
        h = int(rng.integers(1, H + 1)); w = int(rng.integers(1, W + 1))
        crops.append((int(rng.integers(0, H - h + 1)), int(rng.integers(0, W - w + 1)), h, w, int(rng.integers(0, 2))))
    for dtype in (torch.uint8, torch.float32):
        scale, bias = ((1, 1, 1), (0, 0, 0)) if dtype == torch.uint8 else normalize_constants(IMAGENET_MEAN,
                                                                                              IMAGENET_STD)
        got, st = _crop_decode(files, [im.shape[1:] for im in imgs], crops, dtype, scale, bias)
        assert st.tolist() == [0] * len(files)
        for g, im, c in zip(got, imgs, crops):
            ref = _window(im, c)
            if dtype == torch.uint8:
                assert np.array_equal(g, ref), c
            else:
                assert np.abs(g.astype(np.float64) - l3ref.normalize(np.ascontiguousarray(ref), IMAGENET_MEAN,
                                                                     IMAGENET_STD)).max() <= F32_TOL


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("with_crop", [False, True])
def test_hwc_layout_matches_oracle(seed, with_crop):
    """f3: interleaved [h, w, 3] output (L3_DECODE_LAYOUT_HWC), full image or crop + flip, u8 and fp32."""
    rng = np.random.default_rng(70 + seed)
    imgs, files, crops = [], [], []
    for i in range(9):
        H, W = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        N = int(rng.choice([0, 7, 32, 64, 128, 200]))
        im = l3synth.uniform_image(H, W, 90 * seed + i) if i % 2 else l3synth.natural(H, W, 90 * seed + i, 1.0)
        imgs.append(im)
        files.append(l3ref.encode(im, N=N))
        if with_crop:
            h = int(rng.integers(1, H + 1)); w = int(rng.integers(1, W + 1))
            crops.append((int(rng.integers(0, H - h + 1)), int(rng.integers(0, W - w + 1)), h, w,
                          int(rng.integers(0, 2))))
        else:
            crops.append((0, 0, H, W, 0))
    for dtype in (torch.uint8, torch.float32):
        scale, bias = ((1, 1, 1), (0, 0, 0)) if dtype == torch.uint8 else normalize_constants(IMAGENET_MEAN,
                                                                                              IMAGENET_STD)
        got, st = _crop_decode(files, [im.shape[1:] for im in imgs], crops, dtype, scale, bias, layout="hwc",
                               use_crops=with_crop)
        assert st.tolist() == [0] * len(files)
        for g, im, c in zip(got, imgs, crops):
            ref = _window(im, c)
            if dtype == torch.uint8:
                assert np.array_equal(g, ref), c
            else:
                assert np.abs(g.astype(np.float64) - l3ref.normalize(np.ascontiguousarray(ref), IMAGENET_MEAN,
                                                                     IMAGENET_STD)).max() <= F32_TOL


def test_hwc_config3_dense():
    """Dense [n, H, W, 3] u8 output of Cityscapes-shaped images (out_offsets NULL)."""
    imgs = l3synth.make_batch("c3_cityscapes", 3)
    src, offs = pack_files([l3ref.encode(im) for im in imgs])
    out = torch.full((3, 1024, 2048, 3), 0xA5, dtype=torch.uint8, device="cuda")
    dec = BatchDecoder(3)
    sh = torch.tensor([[1024, 2048]] * 3, dtype=torch.int32, device="cuda")
    st, _ = dec.decode(src, offs, sh, out, layout="hwc")
    torch.cuda.synchronize()
    assert st.tolist() == [0, 0, 0]
    got = out.cpu().numpy()
    for i, im in enumerate(imgs):
        assert np.array_equal(got[i], im.transpose(1, 2, 0))


def test_crop_config3_random_crops():
    """Cityscapes-shaped images, training-style random 512x1024 crops with flips."""
    imgs = l3synth.make_batch("c3_cityscapes", 4)
    files = [l3ref.encode(im) for im in imgs]
    crops = [(100, 300, 512, 1024, 0), (0, 0, 512, 1024, 1), (511, 1023, 513, 1025, 1), (37, 901, 512, 1024, 0)]
    got, st = _crop_decode(files, [im.shape[1:] for im in imgs], crops)
    assert st.tolist() == [0] * 4
    for g, im, c in zip(got, imgs, crops):
        assert np.array_equal(g, _window(im, c))


def test_crop_invalid_window_status():
    im = l3synth.natural(40, 50, 1, 1.0)
    f = l3ref.encode(im)
    got, st = _crop_decode([f, f, f], [(40, 50)] * 3, [(0, 0, 40, 50, 0), (30, 0, 11, 50, 0), (0, -1, 4, 4, 0)])
    assert st.tolist() == [0, 1, 1]
    assert np.array_equal(got[0], im)


def test_crop_skips_patches_outside_the_window():
    """A corrupted patch outside the window is never read: the cropped decode stays OK (partial decode)."""
    im = l3synth.natural(256, 256, 3, 1.0)
    f = bytearray(l3ref.encode(im, N=64))
    P = 16
    offs = np.frombuffer(bytes(f[13:13 + 12 * P]), "<u4")
    f[13 + 12 * P + int(offs[15])] &= 0x0F            # k = 0 in unit 15 (bottom-right patch of R)
    got, st = _crop_decode([bytes(f)], [(256, 256)], [(0, 0, 64, 64, 0)])
    assert st.tolist() == [0] and np.array_equal(got[0], im[:, :64, :64])
    got, st = _crop_decode([bytes(f)], [(256, 256)], [(192, 192, 64, 64, 0)])
    assert st.tolist() == [4]


# ------------------------------------------------------------------ f2: ablation decoders

def _ablation_decode(files, imgs, mode):
    from paper_2208_08711_b200 import l3
    src, offs = pack_files(files)
    sizes = [im.size for im in imgs]
    oo = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64), device="cuda")
    out = torch.full((sum(sizes),), 0xA5, dtype=torch.uint8, device="cuda")
    dec = BatchDecoder(len(files))
    sh = torch.tensor([im.shape[1:] for im in imgs], dtype=torch.int32, device="cuda")
    a = dec.args(src, offs, sh, out, out_offsets=oo)
    l3.l3_decode_batch_ablation(a, mode)
    torch.cuda.synchronize()
    flat = out.cpu().numpy()
    got = [flat[o:o + s].reshape(im.shape) for o, s, im in zip(oo.cpu().numpy(), sizes, imgs)]
    return got, dec.status.cpu().numpy()


_ABL_SHAPES = [(70, 133), (300, 260), (64, 64), (1, 5)]
_ABL_NS = [32, 128, 64, 200]


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4, 5])
def test_ablation_decoders_bit_exact(mode):
    imgs = [l3synth.uniform_image(h, w, s) for s, (h, w) in enumerate(_ABL_SHAPES)]
    files = [l3ref.encode(im, N=N) for im, N in zip(imgs, _ABL_NS)]
    got, st = _ablation_decode(files, imgs, mode)
    assert st.tolist() == [0] * len(files)
    for g, im in zip(got, imgs):
        assert np.array_equal(g, im)


@pytest.mark.parametrize("mode", [0, 1, 4, 5])
def test_ablation_original_paeth_variant_bit_exact(mode):
    """The paper's Baseline / +Pixel-wise BD bars decode the original-Paeth variant "L3IP"
    (reading C16); files from the oracle, mixed with custom-Paeth files in one batch."""
    imgs = [l3synth.natural(h, w, s, 1.0) if s % 2 else l3synth.uniform_image(h, w, s)
            for s, (h, w) in enumerate(_ABL_SHAPES + [(129, 257)])]
    Ns = _ABL_NS + [64]
    files = [l3ref.encode_variant(im, N=N) if i != 2 else l3ref.encode(im, N=N)
             for i, (im, N) in enumerate(zip(imgs, Ns))]
    got, st = _ablation_decode(files, imgs, mode)
    assert st.tolist() == [0] * len(files)
    for g, im in zip(got, imgs):
        assert np.array_equal(g, im)


@pytest.mark.parametrize("mode", [2, 3])
def test_ablation_row_parallel_modes_reject_original_paeth(mode):
    imgs = [l3synth.uniform_image(h, w, s) for s, (h, w) in enumerate(_ABL_SHAPES[:2])]
    files = [l3ref.encode_variant(imgs[0], N=32), l3ref.encode(imgs[1], N=128)]
    got, st = _ablation_decode(files, imgs, mode)
    assert st.tolist() == [l3ref.E_UNRECOGNIZED_FORMAT, 0]
    assert np.array_equal(got[1], imgs[1])


def test_hot_path_rejects_original_paeth_variant():
    im = l3synth.uniform_image(40, 50, 1)
    _, st, bad, *_ = gpu_decode([l3ref.encode_variant(im, N=32), l3ref.encode(im, N=32)], [(40, 50)] * 2)
    assert st.tolist() == [l3ref.E_UNRECOGNIZED_FORMAT, 0]


@pytest.mark.parametrize("seed", range(2))
def test_gpu_encoder_original_paeth_byte_identical(seed):
    rng = np.random.default_rng(40 + seed)
    imgs, Ns = [], []
    for i in range(10):
        H, W = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        imgs.append(l3synth.natural(H, W, 10 * seed + i, 1.0) if i % 2 else l3synth.uniform_image(H, W, i))
        Ns.append(int(rng.choice([0, 3, 32, 64, 128, 255])) if H * W < 30000 else 0)
    src, offs = encode_batch(imgs, patch_sizes=Ns, predictor=1)
    o = offs.cpu().numpy()
    buf = src.cpu().numpy()
    for i, (im, N) in enumerate(zip(imgs, Ns)):
        assert buf[o[i]:o[i + 1]].tobytes() == l3ref.encode_variant(im, N=N), (i, im.shape, N)


# ------------------------------------------------------------------ edge cases: sizes and counts

def test_empty_batch_is_a_noop():
    from paper_2208_08711_b200 import l3
    dec = BatchDecoder(4)
    src = torch.zeros(16, dtype=torch.uint8, device="cuda")
    offs = torch.zeros(1, dtype=torch.int64, device="cuda")
    sh = torch.zeros((0, 2), dtype=torch.int32, device="cuda")
    out = torch.zeros(1, dtype=torch.uint8, device="cuda")
    l3.l3_decode_batch(dec.args(src, offs, sh, out))
    torch.cuda.synchronize()


def test_zero_length_and_tiny_files():
    im = l3synth.natural(9, 11, 0, 1.0)
    f = l3ref.encode(im)
    files = [b"", b"L", f, b"L3IF", f[:13], f]
    _, st, bad, _, _, _ = gpu_decode(files, [(9, 11)] * len(files))
    ref = [l3ref.decode(x, exp_shape=(9, 11))[:2] for x in files]
    assert [(int(a), int(b)) for a, b in zip(st, bad)] == [(int(a), int(b)) for a, b in ref]


@pytest.mark.parametrize("n", [1500])
def test_many_images_multi_chunk_parse(n):
    """n > 1024 images: the work decomposition scans in chunks (carry across chunks)."""
    rng = np.random.default_rng(9)
    imgs, files = [], []
    for i in range(n):
        H, W = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        im = l3synth.uniform_image(H, W, i)
        imgs.append(im)
        files.append(l3ref.encode(im, N=int(rng.choice([0, 4, 16, 33, 64, 129]))))
    for wide in (False, True):
        got, st, _, _, _, _ = gpu_decode(files, [im.shape[1:] for im in imgs], wide=wide)
        assert (st == 0).all()
        for g, r in zip(got, imgs):
            assert np.array_equal(g, r)


def test_output_offset_beyond_2_31():
    """Image blocks placed past element 2^31 of a 2.2 GB output: 64-bit output addressing."""
    imgs = [l3synth.natural(130, 260, 1, 2.0), l3synth.natural(64, 200, 2, 2.0)]
    files = [l3ref.encode(im) for im in imgs]
    src, offs = pack_files(files)
    base = (1 << 31) + 12345
    sizes = [im.size for im in imgs]
    out = torch.zeros(base + sum(sizes) + 16, dtype=torch.uint8, device="cuda")
    oo = torch.tensor([base, base + sizes[0]], dtype=torch.int64, device="cuda")
    sh = torch.tensor([im.shape[1:] for im in imgs], dtype=torch.int32, device="cuda")
    dec = BatchDecoder(2)
    st, _ = dec.decode(src, offs, sh, out, out_offsets=oo)
    torch.cuda.synchronize()
    assert st.tolist() == [0, 0]
    for o, s, im in zip([base, base + sizes[0]], sizes, imgs):
        assert np.array_equal(out[o:o + s].cpu().numpy().reshape(im.shape), im)
    assert int(out[:base].count_nonzero()) == 0
    del out
    torch.cuda.empty_cache()


def test_large_single_image():
    """One 8192x6144 image (150 MB raw, 3 x 3072 patches of 128x128)."""
    im = l3synth.natural(6144, 8192, 5, 1.0)
    f = l3ref.encode(im)
    got, st, _, _, _, _ = gpu_decode([f], [im.shape[1:]])
    assert st.tolist() == [0] and np.array_equal(got[0], im)
