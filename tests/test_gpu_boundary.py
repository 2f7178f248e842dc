"""GPU tests of the C-ABI entry points beyond l3_decode_batch, the launch-geometry knob, the
per-unit offset bounds, decoding beside a high-priority compute stream, and bench.py's
multi-rank path (two ranks sharing the one GPU of the box).

Every comparison is against the oracle (oracle/l3ref.c) on the same bytes: pixels bit-exact,
status / bad_unit identical to its sequential decode.
"""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest
import torch

import l3synth
from oracle import l3ref

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2208_08711_b200 import BatchDecoder, l3, pack_files  # noqa: E402
from paper_2208_08711_b200.api import PipelinedLoader  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _units(f):
    W, H, N = struct.unpack("<IIB", f[4:13])
    P = (-(-W // N)) * (-(-H // N))
    data0 = 13 + 12 * P
    return np.frombuffer(f[13:data0], "<u4").astype(np.int64), data0, P


def truncate_inside_unit(f, u):
    """The file cut strictly inside unit u's data (u is not the last unit): every later offset now
    points past the data section."""
    offs, data0, _ = _units(f)
    return f[:data0 + (int(offs[u]) + int(offs[u + 1])) // 2 + 1]


def _faulty_batch(seed=0):
    rng = np.random.default_rng(seed)
    imgs, files = [], []
    for i in range(5):
        H, W = int(rng.integers(30, 200)), int(rng.integers(30, 260))
        im = l3synth.natural(H, W, 10 + i, 2.0)
        imgs.append(im)
        files.append(l3ref.encode(im, N=int(rng.choice([16, 32, 64, 128]))))
    b = bytearray(files[1]); b[0] ^= 0x20; files[1] = bytes(b)                   # magic
    files[2] = files[2][:-9]                                                        # truncated stream
    offs, data0, _ = _units(files[3])
    b = bytearray(files[3]); b[data0 + int(offs[2])] &= 0x0F; files[3] = bytes(b)   # k = 0 in unit 2
    return imgs, files


def _oracle(files, shapes):
    return [l3ref.decode(f, exp_shape=tuple(s)) for f, s in zip(files, shapes)]


def test_load_decode_batch_host_buffers():
    """l3_load_decode_batch: pinned host src -> device, decode, statuses -> pinned host, one call."""
    imgs, files = _faulty_batch(1)
    shapes = [im.shape[1:] for im in imgs]
    n = len(files)
    blob = b"".join(files)
    host_src = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory()
    host_status = torch.full((n,), -7, dtype=torch.int32).pin_memory()
    offs = torch.tensor(np.cumsum([0] + [len(f) for f in files]), dtype=torch.int64, device="cuda")
    dev_src = torch.empty(len(blob) + 16, dtype=torch.uint8, device="cuda")
    sizes = [im.size for im in imgs]
    oo = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64), device="cuda")
    out = torch.full((sum(sizes),), 0xA5, dtype=torch.uint8, device="cuda")
    sh = torch.tensor(np.array(shapes, np.int32), device="cuda")
    dec = BatchDecoder(n)
    stream = torch.cuda.Stream()
    a = dec.args(dev_src, offs, sh, out, out_offsets=oo)
    l3.l3_load_decode_batch(a, host_src, host_status, stream)
    stream.synchronize()
    ref = _oracle(files, shapes)
    assert host_status.tolist() == [r[0] for r in ref]
    assert dec.bad_unit[:n].cpu().tolist() == [r[1] for r in ref]
    flat = out.cpu().numpy()
    for i, (r, o, s) in enumerate(zip(ref, oo.cpu().numpy(), sizes)):
        if r[0] == 0:
            assert np.array_equal(flat[o:o + s].reshape(imgs[i].shape), r[2])


def test_load_decode_batch_argument_errors():
    dec = BatchDecoder(1)
    src = torch.zeros(32, dtype=torch.uint8, device="cuda")
    offs = torch.tensor([0, 16], dtype=torch.int64, device="cuda")
    sh = torch.tensor([[4, 4]], dtype=torch.int32, device="cuda")
    out = torch.zeros(48, dtype=torch.uint8, device="cuda")
    a = dec.args(src, offs, sh, out)
    with pytest.raises(ValueError):            # device tensors where host buffers are required
        l3.l3_load_decode_batch(a, src, dec.status)
    a.src = a.src + 1                           # misaligned device src -> synchronous INVALID_ARGUMENT
    host = torch.zeros(16, dtype=torch.uint8).pin_memory()
    hs = torch.zeros(1, dtype=torch.int32).pin_memory()
    with pytest.raises(l3.L3Error) as e:
        l3.l3_load_decode_batch(a, host, hs)
    assert e.value.status == l3.L3_E_INVALID_ARGUMENT


def _header_variants(f, H, W):
    out = []
    b = bytearray(f); b[3] = ord("X"); out.append((bytes(b), "a1"))                      # magic
    out.append((f[:11], "a1"))                                                          # short header
    _, data0, _ = _units(f)
    out.append((f[:data0 - 3], "a1"))                                                   # offset table cut
    b = bytearray(f); b[4:8] = struct.pack("<I", 0); out.append((bytes(b), "a1"))       # W = 0
    b = bytearray(f); b[12] = 0; out.append((bytes(b), "a1"))                           # N = 0
    b = bytearray(f); b[8:12] = struct.pack("<I", H + 1); out.append((bytes(b), "a1"))  # shape mismatch
    offs, data0, _ = _units(f)
    b = bytearray(f); b[13 + 4 * 2:13 + 4 * 3] = b[13 + 4:13 + 8]; out.append((bytes(b), "unit"))   # offsets
    out.append((f[:-5], "unit"))                                                        # truncated stream
    out.append((f, "ok"))
    return out


def test_parse_batch_header_status():
    """l3_parse_batch (step a1 alone): header-level statuses equal the oracle's; files whose header is
    sound but whose per-unit offsets or streams are bad stay OK (those checks belong to each unit's
    decode); bad_unit is -1 for every file."""
    H, W = 90, 170
    im = l3synth.natural(H, W, 3, 2.0)
    f = l3ref.encode(im, N=32)
    cases = _header_variants(f, H, W)
    files = [c[0] for c in cases]
    src, offs = pack_files(files)
    n = len(files)
    sh = torch.tensor([[H, W]] * n, dtype=torch.int32, device="cuda")
    out = torch.zeros(3 * H * W * n, dtype=torch.uint8, device="cuda")
    dec = BatchDecoder(n)
    dec.status.fill_(-9)
    dec.bad_unit.fill_(-9)
    l3.l3_parse_batch(dec.args(src, offs, sh, out))
    torch.cuda.synchronize()
    st = dec.status[:n].cpu().tolist()
    ref = _oracle(files, [(H, W)] * n)
    for (fi, kind), s, r in zip(cases, st, ref):
        if kind == "a1":
            assert s == r[0] and s in (l3ref.E_UNRECOGNIZED_FORMAT, l3ref.E_CORRUPT_HEADER), (kind, s, r[0])
        else:
            assert s == 0, (kind, s)
    assert dec.bad_unit[:n].cpu().tolist() == [-1] * n
    assert int(out.count_nonzero()) == 0                        # a1 decodes nothing
    # the workspace stays valid for a decode after the parse-only call
    st2, bad2 = dec.decode(src, offs, sh, out, out_offsets=torch.arange(n, device="cuda") * 3 * H * W)
    torch.cuda.synchronize()
    assert [(int(a), int(b)) for a, b in zip(st2.cpu(), bad2.cpu())] == [(r[0], r[1]) for r in ref]


@pytest.mark.parametrize("variant", ["u8", "u8wide", "f32", "hwc_u8", "hwc_f32"])
def test_truncated_inside_unit_last_file(variant):
    """A file cut inside a unit's data, placed LAST in an exactly-sized source buffer: the unit's
    next offset points past the data section, so the oracle says CORRUPT_HEADER and the decoder must
    say the same without reading past the file."""
    imgs = [l3synth.natural(130, 300, 1, 2.0), l3synth.natural(200, 260, 2, 2.0), l3synth.natural(96, 160, 3, 2.0)]
    Ns = [64, 128, 32]
    files = [l3ref.encode(im, N=N) for im, N in zip(imgs, Ns)]
    files.append(truncate_inside_unit(files[1], 1))
    files.append(truncate_inside_unit(files[2], 3))
    imgs += [imgs[1], imgs[2]]
    shapes = [im.shape[1:] for im in imgs]
    ref = _oracle(files, shapes)
    assert [r[0] for r in ref] == [0, 0, 0, l3ref.E_CORRUPT_HEADER, l3ref.E_CORRUPT_HEADER]
    src, offs = pack_files(files)
    assert src.numel() == int(offs[-1])                         # no slack after the last file
    n = len(files)
    sizes = [im.size for im in imgs]
    oo = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64), device="cuda")
    dtype = torch.float32 if "f32" in variant else torch.uint8
    out = torch.zeros(sum(sizes), dtype=dtype, device="cuda")
    sh = torch.tensor(np.array(shapes, np.int32), device="cuda")
    dec = BatchDecoder(n)
    st, bad = dec.decode(src, offs, sh, out, out_offsets=oo, wide=(variant == "u8wide"),
                         layout="hwc" if variant.startswith("hwc") else "chw")
    torch.cuda.synchronize()
    assert [(int(a), int(b)) for a, b in zip(st.cpu(), bad.cpu())] == [(r[0], r[1]) for r in ref]


def test_crop_touching_truncated_unit_but_not_the_next():
    """Partial decode whose window touches unit u (the file is cut inside it) but not unit u+1: the
    decoder still sees that u's byte range ends past the file (CORRUPT_HEADER, as the oracle)."""
    H, W, N = 256, 256, 64
    im = l3synth.natural(H, W, 5, 2.0)
    f = l3ref.encode(im, N=N)
    _, _, P = _units(f)
    u = 2 * P + 5                                  # B channel, patch 5 = (px 1, py 1); unit u+1 = patch 6
    tf = truncate_inside_unit(f, u)
    assert l3ref.decode(tf, exp_shape=(H, W))[0] == l3ref.E_CORRUPT_HEADER
    src, offs = pack_files([tf])
    crops = torch.tensor([[64 + 3, 64 + 5, 40, 50, 1]], dtype=torch.int32, device="cuda")   # inside patch 5
    sh = torch.tensor([[H, W]], dtype=torch.int32, device="cuda")
    dec = BatchDecoder(1)
    for dtype in (torch.uint8, torch.float32):
        for layout in ("chw", "hwc"):
            out = torch.zeros(3 * 40 * 50, dtype=dtype, device="cuda")
            st, _ = dec.decode(src, offs, sh, out, crops=crops, layout=layout)
            torch.cuda.synchronize()
            assert int(st[0]) == l3ref.E_CORRUPT_HEADER, (dtype, layout)


@pytest.mark.parametrize("max_ctas", [1, 2, 7, 148, 5000, 0])
def test_max_ctas_any_grid_decodes(max_ctas):
    """l3_decode_args.max_ctas caps the persistent grid (to leave SMs to compute); any cap decodes the
    same pixels and statuses, including the a1 election and a7 finish with a single CTA."""
    imgs, files = _faulty_batch(2)
    imgs.append(l3synth.natural(1024, 2048, 7, 0.48))
    files.append(l3ref.encode(imgs[-1]))
    shapes = [im.shape[1:] for im in imgs]
    ref = _oracle(files, shapes)
    src, offs = pack_files(files)
    n = len(files)
    sizes = [im.size for im in imgs]
    oo_np = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    oo = torch.tensor(oo_np, device="cuda")
    sh = torch.tensor(np.array(shapes, np.int32), device="cuda")
    dec = BatchDecoder(n)
    for dtype, wide, layout in ((torch.uint8, False, "chw"), (torch.uint8, True, "chw"), (torch.float32, False, "chw"),
                                (torch.uint8, False, "hwc")):
        out = torch.zeros(sum(sizes), dtype=dtype, device="cuda")
        st, bad = dec.decode(src, offs, sh, out, out_offsets=oo, wide=wide, layout=layout, max_ctas=max_ctas)
        torch.cuda.synchronize()
        assert [(int(a), int(b)) for a, b in zip(st.cpu(), bad.cpu())] == [(r[0], r[1]) for r in ref]
        if dtype == torch.uint8:
            flat = out.cpu().numpy()
            for i, r in enumerate(ref):
                if r[0] == 0:
                    g = flat[oo_np[i]:oo_np[i] + sizes[i]]
                    g = g.reshape(imgs[i].shape) if layout == "chw" else \
                        g.reshape(imgs[i].shape[1], imgs[i].shape[2], 3).transpose(2, 0, 1)
                    assert np.array_equal(g, r[2]), (max_ctas, wide, layout, i)


def test_decode_beside_high_priority_compute():
    """the decoder runs on a low-priority stream while a long bf16 GEMM loop holds the
    SMs from a high-priority stream. The persistent decode grid cannot be fully resident while the GEMMs
    run; the first CTA to arrive parses (a1 election), so the launch completes whatever CTAs get SMs
    first, and the pixels are exact."""
    imgs = l3synth.make_batch("c3_cityscapes", 6)
    files = [l3ref.encode(im) for im in imgs]
    src, offs = pack_files(files)
    n = len(files)
    sh = torch.tensor([[1024, 2048]] * n, dtype=torch.int32, device="cuda")
    lo, hi = torch.cuda.Stream.priority_range()
    cs = torch.cuda.Stream(priority=hi)
    ds = torch.cuda.Stream(priority=lo)
    A = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
    B = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
    C = torch.empty_like(A)
    ref_c = torch.matmul(A, B)
    torch.cuda.synchronize()
    for max_ctas in (0, 64):
        dec = BatchDecoder(n)
        outs = [torch.full((n, 3, 1024, 2048), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(3)]
        with torch.cuda.stream(cs):
            for _ in range(30):
                torch.matmul(A, B, out=C)
        for o in outs:       # enqueued while the GEMMs are running
            dec.decode(src, offs, sh, o, stream=ds, max_ctas=max_ctas)
        ds.synchronize()
        cs.synchronize()
        assert dec.status[:n].cpu().tolist() == [0] * n
        for o in outs:
            got = o.cpu().numpy()
            for i in range(n):
                assert np.array_equal(got[i], imgs[i]), (max_ctas, i)
        assert torch.allclose(C.float(), ref_c.float(), rtol=1e-2, atol=1e-2)


def test_pipelined_loader_matches_direct_decode():
    """f1 loader: every batch is one l3_load_decode_batch call (host buffers) on alternating
    low-priority streams; same pixels / statuses as the oracle, per-ticket statuses kept."""
    imgs = [l3synth.natural(200, 300, s, 2.0) for s in range(6)]
    files = [l3ref.encode(im) for im in imgs]
    bad = bytearray(files[4]); bad[13 + 12 * 70 + 40] &= 0x0F   # changes pixels (still a valid stream)
    off5 = int.from_bytes(bad[13 + 4 * 5:17 + 4 * 5], "little")
    bad[13 + 12 * 70 + off5] &= 0x0F                              # unit 5, row 0: k = 0 -> CORRUPT_STREAM
    files_b = [files[:3], [files[3], bytes(bad), files[5]]]
    # the oracle's decode of every file (the injected byte may change pixels without a stream error)
    ref_dec = [[l3ref.decode(f, exp_shape=(200, 300)) for f in b] for b in files_b]
    ref_st = [[r[0] for r in rb] for rb in ref_dec]
    loader = PipelinedLoader(3, max(sum(map(len, b)) for b in files_b), depth=2)
    hs = torch.full((4, 3), -1, dtype=torch.int32).pin_memory()
    outs = []
    for k, b in enumerate(files_b + files_b):
        offs = torch.tensor(np.cumsum([0] + [len(f) for f in b]), dtype=torch.int64, device="cuda")
        host = torch.from_numpy(np.frombuffer(b"".join(b), np.uint8).copy()).pin_memory()
        sh = torch.tensor([[200, 300]] * len(b), dtype=torch.int32, device="cuda")
        out = torch.empty((len(b), 3, 200, 300), dtype=torch.uint8, device="cuda")
        loader.submit(host, offs, sh, out, host_status=hs[k])
        outs.append(out)
    torch.cuda.synchronize()
    assert ref_st[1][1] == l3ref.E_CORRUPT_STREAM
    for k in range(4):
        assert hs[k].tolist() == ref_st[k % 2]
    for k, out in enumerate(outs):
        for i in range(3):
            if ref_st[k % 2][i] == 0:
                assert np.array_equal(out[i].cpu().numpy(), ref_dec[k % 2][i][2]), (k, i)
    # internal status slots: waiting for a ticket whose slot was reused raises
    t0 = loader.submit(host, offs, sh, outs[-1])
    loader.submit(host, offs, sh, outs[-1])
    loader.submit(host, offs, sh, outs[-1])
    with pytest.raises(RuntimeError):
        loader.wait(t0)


def test_bench_two_ranks_share_device():
    """bench.py's multi-rank path (init_process_group, barriers, max-over-ranks timing, aggregate line)
    run as 2 ranks on the one GPU (gloo for the plumbing): one JSON line, n_gpus 2, statuses OK, the
    aggregate roofline fraction of SURVEY §8(e)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2", "--steps", "5",
           "--warmup", "3", "--e2e-steps", "3", "--share-device", "--dist-backend", "gloo", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["status_ok"] and d["self_check"]
    assert d["config"]["global_batch"] == 64 and d["steps"] == 5
    roof = d["roofline"]
    assert 0 < roof["aggregate_frac"] and roof["aggregate_alg_bytes"] > roof["alg_bytes_per_launch"]
    assert d["e2e"]["value"] > 0 and d["value"] > 0


def test_decode_in_cuda_graph():
    """l3_decode_batch captured in a CUDA graph (its two launches and their programmatic dependency
    become graph nodes) and replayed on new inputs copied into the captured buffers: pixels and
    statuses equal the oracle's on every replay."""
    imgs = [l3synth.natural(200, 300, 30 + i, 2.0) for i in range(4)]
    files = [l3ref.encode(im) for im in imgs]
    other = [l3synth.natural(200, 300, 40 + i, 2.0) for i in range(4)]
    files2 = [l3ref.encode(im) for im in other]
    cap = max(sum(map(len, files)), sum(map(len, files2))) + 16
    src = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    offs = torch.zeros(5, dtype=torch.int64, device="cuda")
    shapes = torch.tensor([[200, 300]] * 4, dtype=torch.int32, device="cuda")
    out = torch.zeros((4, 3, 200, 300), dtype=torch.uint8, device="cuda")
    dec = BatchDecoder(4)
    s = torch.cuda.Stream()

    def load(fs):
        o = np.cumsum([0] + [len(f) for f in fs])
        src[:int(o[-1])].copy_(torch.from_numpy(np.frombuffer(b"".join(fs), np.uint8).copy()))
        offs.copy_(torch.from_numpy(o.astype(np.int64)))

    load(files)
    torch.cuda.synchronize()
    a = dec.args(src, offs, shapes, out)
    with torch.cuda.stream(s):
        l3.l3_decode_batch(a, s)   # warm up outside the capture
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        l3.l3_decode_batch(a, s)
    for fs, ref in ((files, imgs), (files2, other), (files, imgs)):
        load(fs)
        out.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert dec.status[:4].cpu().tolist() == [0] * 4
        got = out.cpu().numpy()
        for i in range(4):
            assert np.array_equal(got[i], ref[i]), i
