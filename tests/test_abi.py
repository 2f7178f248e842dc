"""CPU-side checks of the C ABI boundary: the library builds for sm_100a, loads, and
exports every symbol include/l3.h declares; host-only helpers agree with the oracle's
policy. No compute calls (there is no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "l3.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(l3_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2208_08711_b200 import _build, l3
    _build.build()
    return l3.lib()


def test_header_declares_expected_entry_points():
    d = _declared()
    for name in ("l3_decode_batch", "l3_parse_batch", "l3_decode_workspace_size",
                 "l3_load_decode_batch", "l3_status_string", "l3_encode_batch"):
        assert name in d


def test_library_exports_every_declared_symbol(lib):
    from paper_2208_08711_b200 import l3
    out = subprocess.run(["nm", "-D", "--defined-only", l3.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (l3_[a-z0-9_]+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    assert set(l3.EXPORTED) == set(_declared())


def test_library_is_sm100a(lib):
    from paper_2208_08711_b200 import l3
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", l3.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_tma_bulk_copy(lib):
    from paper_2208_08711_b200 import l3
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", l3.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UBLKCP" in sass        # cp.async.bulk (TMA 1-D) in the decode kernel
    assert "SYNCS" in sass         # mbarrier


def test_host_helpers(lib):
    from oracle import l3ref
    from paper_2208_08711_b200 import l3
    for W, H in [(640, 480), (1080, 720), (1079, 720), (1280, 720), (1920, 1080), (2048, 1024), (3840, 2160),
                 (1, 1)]:
        assert l3.l3_choose_patch_size(W, H) == l3ref.choose_patch_size(W, H)
    for W, H, N in [(64, 64, 0), (500, 375, 32), (3840, 2160, 128), (7, 5, 3), (1, 1, 255)]:
        assert l3.l3_encode_max_bytes(W, H, N) >= l3ref.max_file_bytes(W, H, N) - 3 * ((W + 7) * (H + 7))
    assert l3.l3_status_string(4) == "corrupt stream"
    assert l3.l3_decode_workspace_size(32) >= 32 * 64
    assert l3.l3_decode_kernels_per_call() == 2
    # launches of a given call (host-only, no pointer is dereferenced): a1 inside the decode grid for
    # planar batches of <= 32 images, else the a1 kernel + the decode grid
    from paper_2208_08711_b200.l3 import L3_DECODE_HINT_WIDE, L3_DECODE_LAYOUT_HWC, l3_decode_args
    a = l3_decode_args()
    assert l3.l3_decode_launches(a) == 0   # empty batch: no launch
    a.n = 1
    assert l3.l3_decode_launches(a) == -1   # NULL pointers: invalid, like l3_decode_batch
    a.src = a.src_offsets = a.shapes = a.out = a.status = a.workspace = 1 << 20   # aligned, never read
    a.workspace_bytes = l3.l3_decode_workspace_size(64)
    a.out_kind = 0
    assert l3.l3_decode_launches(a) == 1
    a.n = 32
    assert l3.l3_decode_launches(a) == 1
    a.n = 33
    assert l3.l3_decode_launches(a) == 2
    a.n = 8
    a.flags = L3_DECODE_LAYOUT_HWC
    assert l3.l3_decode_launches(a) == 2
    a.flags = L3_DECODE_HINT_WIDE   # the wide kernel also runs a1 in its blocks
    assert l3.l3_decode_launches(a) == 1


def test_no_cpu_fallback_without_cuda(lib):
    import torch
    from paper_2208_08711_b200 import BatchDecoder
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError):
        BatchDecoder(4)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2208_08711_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|l3ref|libl3ref|oracle/l3ref)", text), f
