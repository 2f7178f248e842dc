"""Thin ctypes binding of include/l3.h (argument marshalling only).

Every function here has the name of the C entry point it calls and does nothing
but check/convert arguments: all decode work runs in the sm_100a kernels of
``libl3_b200.so``. There is no CPU fallback — if the library or a CUDA device
is missing these functions raise.

torch is used for device memory and streams only (``data_ptr()``,
``torch.cuda.current_stream().cuda_stream``).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("L3_B200_LIB_OVERRIDE") or os.path.join(_PKG, "libl3_b200.so")   # override: dev A/B only

L3_OK, L3_E_INVALID_ARGUMENT, L3_E_UNRECOGNIZED_FORMAT, L3_E_CORRUPT_HEADER, L3_E_CORRUPT_STREAM, \
    L3_E_TRUNCATED_STREAM, L3_E_CUDA = range(7)
L3_OUT_U8, L3_OUT_F32 = 0, 1

STATUS_NAMES = {L3_OK: "OK", L3_E_INVALID_ARGUMENT: "INVALID_ARGUMENT",
                L3_E_UNRECOGNIZED_FORMAT: "UNRECOGNIZED_FORMAT", L3_E_CORRUPT_HEADER: "CORRUPT_HEADER",
                L3_E_CORRUPT_STREAM: "CORRUPT_STREAM", L3_E_TRUNCATED_STREAM: "TRUNCATED_STREAM",
                L3_E_CUDA: "CUDA"}


class l3_decode_args(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_void_p),
        ("src_offsets", ctypes.c_void_p),
        ("shapes", ctypes.c_void_p),
        ("n", ctypes.c_int32),
        ("out_kind", ctypes.c_int32),
        ("out", ctypes.c_void_p),
        ("out_offsets", ctypes.c_void_p),
        ("scale", ctypes.c_float * 3),
        ("bias", ctypes.c_float * 3),
        ("status", ctypes.c_void_p),
        ("bad_unit", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_uint64),
        ("flags", ctypes.c_uint32),
        ("max_ctas", ctypes.c_uint32),
        ("crops", ctypes.c_void_p),
    ]


L3_DECODE_HINT_WIDE = 1
L3_DECODE_LAYOUT_HWC = 2


class l3_encode_args(ctypes.Structure):
    _fields_ = [
        ("images", ctypes.c_void_p),
        ("img_offsets_host", ctypes.c_void_p),
        ("shapes_host", ctypes.c_void_p),
        ("n_host", ctypes.c_void_p),
        ("n", ctypes.c_int32),
        ("dst", ctypes.c_void_p),
        ("dst_capacity", ctypes.c_uint64),
        ("dst_offsets", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_uint64),
        ("predictor", ctypes.c_int32),
    ]


_lock = threading.Lock()
_lib = None


class L3Error(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(status, status)}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libl3_b200.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            P = ctypes.POINTER
            for name in ("l3_decode_batch", "l3_parse_batch"):
                getattr(L, name).argtypes = [P(l3_decode_args), ctypes.c_void_p]
                getattr(L, name).restype = ctypes.c_int
            L.l3_load_decode_batch.argtypes = [P(l3_decode_args), ctypes.c_void_p, ctypes.c_uint64,
                                               ctypes.c_void_p, ctypes.c_void_p]
            L.l3_load_decode_batch.restype = ctypes.c_int
            L.l3_decode_workspace_size.argtypes = [ctypes.c_int32]
            L.l3_decode_workspace_size.restype = ctypes.c_uint64
            L.l3_decode_kernels_per_call.argtypes = []
            L.l3_decode_kernels_per_call.restype = ctypes.c_int32
            L.l3_decode_launches.argtypes = [ctypes.c_void_p]
            L.l3_decode_launches.restype = ctypes.c_int32
            L.l3_decode_batch_ablation.argtypes = [P(l3_decode_args), ctypes.c_int32, ctypes.c_void_p]
            L.l3_decode_batch_ablation.restype = ctypes.c_int
            L.l3_selftest_paeth.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
            L.l3_selftest_paeth.restype = ctypes.c_int
            L.l3_selftest_paeth4.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
            L.l3_selftest_paeth4.restype = ctypes.c_int
            L.l3_selftest_paeth_h2.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
            L.l3_selftest_paeth_h2.restype = ctypes.c_int
            L.l3_status_string.argtypes = [ctypes.c_int32]
            L.l3_status_string.restype = ctypes.c_char_p
            L.l3_choose_patch_size.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
            L.l3_choose_patch_size.restype = ctypes.c_int32
            L.l3_encode_max_bytes.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int32]
            L.l3_encode_max_bytes.restype = ctypes.c_uint64
            L.l3_encode_workspace_size.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
            L.l3_encode_workspace_size.restype = ctypes.c_uint64
            L.l3_encode_batch.argtypes = [P(l3_encode_args), ctypes.c_void_p]
            L.l3_encode_batch.restype = ctypes.c_int
            _lib = L
    return _lib


EXPORTED = ("l3_decode_workspace_size", "l3_decode_batch", "l3_parse_batch",
            "l3_load_decode_batch", "l3_decode_kernels_per_call", "l3_decode_launches", "l3_status_string",
            "l3_choose_patch_size",
            "l3_encode_max_bytes", "l3_encode_workspace_size", "l3_encode_batch", "l3_selftest_paeth",
            "l3_selftest_paeth4", "l3_selftest_paeth_h2", "l3_decode_batch_ablation")


def _dev_ptr(t: torch.Tensor | None, name: str, dtype=None) -> int:
    if t is None:
        return 0
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def make_decode_args(src, src_offsets, shapes, out, status, workspace, *, out_offsets=None, bad_unit=None,
                     scale=(1.0, 1.0, 1.0), bias=(0.0, 0.0, 0.0), flags=0, crops=None,
                     max_ctas=0) -> l3_decode_args:
    a = l3_decode_args()
    a.src = _dev_ptr(src, "src", torch.uint8)
    a.src_offsets = _dev_ptr(src_offsets, "src_offsets", torch.int64)
    a.shapes = _dev_ptr(shapes, "shapes", torch.int32)
    a.n = int(shapes.shape[0])
    if out.dtype == torch.uint8:
        a.out_kind = L3_OUT_U8
    elif out.dtype == torch.float32:
        a.out_kind = L3_OUT_F32
    else:
        raise ValueError("out must be uint8 or float32")
    a.out = _dev_ptr(out, "out")
    a.out_offsets = _dev_ptr(out_offsets, "out_offsets", torch.int64)
    a.scale = (ctypes.c_float * 3)(*[float(x) for x in scale])
    a.bias = (ctypes.c_float * 3)(*[float(x) for x in bias])
    a.status = _dev_ptr(status, "status", torch.int32)
    a.bad_unit = _dev_ptr(bad_unit, "bad_unit", torch.int32)
    a.workspace = _dev_ptr(workspace, "workspace")
    a.workspace_bytes = workspace.numel() * workspace.element_size()
    a.flags = int(flags)
    a.crops = _dev_ptr(crops, "crops", torch.int32)
    a.max_ctas = int(max_ctas)
    return a


def _check(fn: str, st: int) -> None:
    if st != L3_OK:
        raise L3Error(fn, st)


def l3_decode_workspace_size(n: int) -> int:
    return int(lib().l3_decode_workspace_size(n))


def l3_decode_kernels_per_call() -> int:
    return int(lib().l3_decode_kernels_per_call())


def l3_decode_launches(args: l3_decode_args) -> int:
    return int(lib().l3_decode_launches(ctypes.byref(args)))


def l3_decode_batch(args: l3_decode_args, stream=None) -> None:
    _check("l3_decode_batch", lib().l3_decode_batch(ctypes.byref(args), _stream(stream)))


def l3_parse_batch(args: l3_decode_args, stream=None) -> None:
    _check("l3_parse_batch", lib().l3_parse_batch(ctypes.byref(args), _stream(stream)))


def l3_load_decode_batch(args: l3_decode_args, host_src: torch.Tensor, host_status: torch.Tensor,
                         stream=None) -> None:
    if host_src.is_cuda or host_status.is_cuda:
        raise ValueError("host_src / host_status must be (pinned) host tensors")
    _check("l3_load_decode_batch",
           lib().l3_load_decode_batch(ctypes.byref(args), host_src.data_ptr(), host_src.numel(),
                                      host_status.data_ptr(), _stream(stream)))


def l3_decode_batch_ablation(args: l3_decode_args, mode: int, stream=None) -> None:
    _check("l3_decode_batch_ablation", lib().l3_decode_batch_ablation(ctypes.byref(args), int(mode), _stream(stream)))


def l3_selftest_paeth(out: torch.Tensor, stream=None) -> None:
    if out.numel() < (1 << 24):
        raise ValueError("out needs 2^24 bytes")
    _check("l3_selftest_paeth", lib().l3_selftest_paeth(_dev_ptr(out, "out", torch.uint8), _stream(stream)))


def l3_selftest_paeth4(out: torch.Tensor, stream=None) -> None:
    if out.numel() < (4 << 24):
        raise ValueError("out needs 4 * 2^24 bytes")
    _check("l3_selftest_paeth4", lib().l3_selftest_paeth4(_dev_ptr(out, "out", torch.uint8), _stream(stream)))


def l3_selftest_paeth_h2(out: torch.Tensor, stream=None) -> None:
    if out.numel() < (1 << 24):
        raise ValueError("out needs 2^24 bytes")
    _check("l3_selftest_paeth_h2", lib().l3_selftest_paeth_h2(_dev_ptr(out, "out", torch.uint8), _stream(stream)))


def l3_status_string(status: int) -> str:
    return lib().l3_status_string(status).decode()


def l3_choose_patch_size(W: int, H: int) -> int:
    return int(lib().l3_choose_patch_size(W, H))


def l3_encode_max_bytes(W: int, H: int, N: int = 0) -> int:
    return int(lib().l3_encode_max_bytes(W, H, N))


def l3_encode_workspace_size(shapes_host, n_host=None) -> int:
    import numpy as np
    sh = np.ascontiguousarray(shapes_host, np.int32)
    nh = None if n_host is None else np.ascontiguousarray(n_host, np.int32)
    return int(lib().l3_encode_workspace_size(sh.ctypes.data, 0 if nh is None else nh.ctypes.data, len(sh)))


def l3_encode_batch(images: torch.Tensor, img_offsets_host, shapes_host, n_host, dst: torch.Tensor,
                    dst_offsets: torch.Tensor, workspace: torch.Tensor, stream=None, predictor: int = 0) -> None:
    import numpy as np
    io = np.ascontiguousarray(img_offsets_host, np.uint64)
    sh = np.ascontiguousarray(shapes_host, np.int32)
    nh = None if n_host is None else np.ascontiguousarray(n_host, np.int32)
    a = l3_encode_args()
    a.images = _dev_ptr(images, "images", torch.uint8)
    a.img_offsets_host = io.ctypes.data
    a.shapes_host = sh.ctypes.data
    a.n_host = 0 if nh is None else nh.ctypes.data
    a.n = len(sh)
    a.dst = _dev_ptr(dst, "dst", torch.uint8)
    a.dst_capacity = dst.numel()
    a.dst_offsets = _dev_ptr(dst_offsets, "dst_offsets", torch.int64)
    a.workspace = _dev_ptr(workspace, "workspace")
    a.workspace_bytes = workspace.numel() * workspace.element_size()
    a.predictor = predictor
    _check("l3_encode_batch", lib().l3_encode_batch(ctypes.byref(a), _stream(stream)))
