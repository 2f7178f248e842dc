"""ctypes binding of the C oracle (oracle/l3ref.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package. Builds ``oracle/libl3ref.so`` with gcc on first use if it is missing.

Status codes are restated here, independently of include/l3.h.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libl3ref.so")

OK, E_INVALID_ARGUMENT, E_UNRECOGNIZED_FORMAT, E_CORRUPT_HEADER, E_CORRUPT_STREAM, E_TRUNCATED_STREAM = range(6)
BASE_SIGNED, BASE_UNSIGNED = 0, 1

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math, so fmaf/double are IEEE)."""
    src = os.path.join(HERE, "l3ref.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-pthread", "-fno-fast-math",
             "-ffp-contract=off", "-o", tmp, src])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(LIB_PATH)
            u8p = ctypes.POINTER(ctypes.c_uint8)
            L.l3ref_predict.argtypes = [ctypes.c_int] * 3
            L.l3ref_predict.restype = ctypes.c_int
            L.l3ref_predict_many.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint64, ctypes.c_void_p]
            L.l3ref_predict_many.restype = None
            L.l3ref_predict_png_many.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint64, ctypes.c_void_p]
            L.l3ref_predict_png_many.restype = None
            L.l3ref_predict_png.argtypes = [ctypes.c_int] * 3
            L.l3ref_predict_png.restype = ctypes.c_int
            L.l3ref_encode_image_variant.argtypes = [u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                                     ctypes.c_int, u8p, ctypes.c_uint64]
            L.l3ref_encode_image_variant.restype = ctypes.c_uint64
            L.l3ref_decode_image_variant.argtypes = [u8p, ctypes.c_uint64, u8p, ctypes.c_uint64,
                                                     ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
            L.l3ref_decode_image_variant.restype = ctypes.c_int
            L.l3ref_choose_patch_size.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
            L.l3ref_choose_patch_size.restype = ctypes.c_int
            L.l3ref_bd_encode_row.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), u8p]
            L.l3ref_bd_encode_row.restype = None
            L.l3ref_max_file_bytes.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int]
            L.l3ref_max_file_bytes.restype = ctypes.c_uint64
            L.l3ref_encode_image.argtypes = [u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, u8p, ctypes.c_uint64]
            L.l3ref_encode_image.restype = ctypes.c_uint64
            L.l3ref_decode_image.argtypes = [u8p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, u8p,
                                             ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64),
                                             ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                             ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_uint64)]
            L.l3ref_decode_image.restype = ctypes.c_int
            L.l3ref_decode_batch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_int]
            L.l3ref_decode_batch.restype = None
            L.l3ref_normalize.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]
            L.l3ref_normalize.restype = None
            _lib = L
    return _lib


def _u8(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def predict(tl: int, t: int, tr: int) -> int:
    return lib().l3ref_predict(tl, t, tr)


def predict_many(tl: np.ndarray, t: np.ndarray, tr: np.ndarray) -> np.ndarray:
    tl, t, tr = (np.ascontiguousarray(a, np.uint8) for a in (tl, t, tr))
    out = np.zeros(len(t), np.uint8)
    lib().l3ref_predict_many(tl.ctypes.data, t.ctypes.data, tr.ctypes.data, len(t), out.ctypes.data)
    return out


def predict_png_many(a: np.ndarray, b: np.ndarray, c: np.ndarray) -> np.ndarray:
    a, b, c = (np.ascontiguousarray(x, np.uint8) for x in (a, b, c))
    out = np.zeros(len(a), np.uint8)
    lib().l3ref_predict_png_many(a.ctypes.data, b.ctypes.data, c.ctypes.data, len(a), out.ctypes.data)
    return out


def choose_patch_size(W: int, H: int) -> int:
    return lib().l3ref_choose_patch_size(W, H)


def bd_encode_row(res, first_row: bool, base_rule: int = BASE_SIGNED, k_extra: int = 0):
    res = np.ascontiguousarray(res, dtype=np.uint8)
    d = np.zeros(len(res), np.uint8)
    k, b = ctypes.c_int(), ctypes.c_int()
    lib().l3ref_bd_encode_row(_u8(res), len(res), int(first_row), base_rule, k_extra,
                              ctypes.byref(k), ctypes.byref(b), _u8(d))
    return k.value, b.value, d


def max_file_bytes(W: int, H: int, N: int = 0) -> int:
    return int(lib().l3ref_max_file_bytes(W, H, N))


def encode(planar: np.ndarray, N: int = 0, base_rule: int = BASE_SIGNED, k_extra: int = 0) -> bytes:
    """planar: uint8 [3, H, W]. Returns the L3 file bytes."""
    planar = np.ascontiguousarray(planar, dtype=np.uint8)
    assert planar.ndim == 3 and planar.shape[0] == 3
    _, H, W = planar.shape
    cap = max_file_bytes(W, H, N)
    out = np.zeros(cap, np.uint8)
    n = lib().l3ref_encode_image(_u8(planar), W, H, N, base_rule, k_extra, _u8(out), cap)
    if n == 0:
        raise ValueError("l3ref_encode_image failed")
    return out[:n].tobytes()


def predict_png(a: int, b: int, c: int) -> int:
    return lib().l3ref_predict_png(a, b, c)


def encode_variant(planar: np.ndarray, N: int = 0, predictor: int = 1) -> bytes:
    """Ablation format variant (f2): predictor 1 = original Paeth (magic "L3IP")."""
    planar = np.ascontiguousarray(planar, dtype=np.uint8)
    _, H, W = planar.shape
    cap = max_file_bytes(W, H, N)
    out = np.zeros(cap, np.uint8)
    n = lib().l3ref_encode_image_variant(_u8(planar), W, H, N, predictor, _u8(out), cap)
    if n == 0:
        raise ValueError("l3ref_encode_image_variant failed")
    return out[:n].tobytes()


def decode_variant(data: bytes, shape):
    """Decode an L3IF or L3IP file of known shape (H, W). Returns (status, planar)."""
    H, W = shape
    buf = np.frombuffer(data, np.uint8)
    out = np.zeros((3, H, W), np.uint8)
    w, h = ctypes.c_uint32(), ctypes.c_uint32()
    st = lib().l3ref_decode_image_variant(_u8(buf), len(data), _u8(out), out.size, ctypes.byref(w), ctypes.byref(h))
    return st, out


def decode(data: bytes, exp_shape=None):
    """Sequential decode of one file. Returns (status, bad_unit, planar or None, (W, H, N, P))."""
    buf = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
    W, H, N, P = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_int(), ctypes.c_uint64()
    bad = ctypes.c_int64()
    eH, eW = (0, 0) if exp_shape is None else exp_shape
    # first pass: read the header to size the output
    st = lib().l3ref_decode_image(_u8(buf), len(data), eW, eH, None, 0, ctypes.byref(bad),
                                  ctypes.byref(W), ctypes.byref(H), ctypes.byref(N), ctypes.byref(P))
    if st != E_INVALID_ARGUMENT:
        return st, bad.value, None, (W.value, H.value, N.value, P.value)
    out = np.zeros((3, H.value, W.value), np.uint8)
    st = lib().l3ref_decode_image(_u8(buf), len(data), eW, eH, _u8(out), out.size, ctypes.byref(bad),
                                  ctypes.byref(W), ctypes.byref(H), ctypes.byref(N), ctypes.byref(P))
    return st, bad.value, out, (W.value, H.value, N.value, P.value)


def decode_batch(src: np.ndarray, src_offsets: np.ndarray, shapes: np.ndarray, threads: int = 1):
    """Batch decode. shapes: int32 [n, 2] (H, W). Returns (list of planar arrays, status, bad_unit)."""
    src = np.ascontiguousarray(src, np.uint8)
    src_offsets = np.ascontiguousarray(src_offsets, np.uint64)
    shapes = np.ascontiguousarray(shapes, np.int32)
    n = len(shapes)
    sizes = 3 * shapes[:, 0].astype(np.uint64) * shapes[:, 1].astype(np.uint64)
    out_offsets = np.zeros(n, np.uint64)
    if n > 1:
        out_offsets[1:] = np.cumsum(sizes)[:-1]
    out = np.zeros(int(sizes.sum()) if n else 1, np.uint8)
    status = np.zeros(n, np.int32)
    bad = np.zeros(n, np.int32)
    lib().l3ref_decode_batch(src.ctypes.data, src_offsets.ctypes.data, shapes.ctypes.data, n,
                             out.ctypes.data, out_offsets.ctypes.data, status.ctypes.data, bad.ctypes.data,
                             threads)
    imgs = [out[int(o):int(o) + int(s)].reshape(3, int(h), int(w))
            for o, s, (h, w) in zip(out_offsets, sizes, shapes)]
    return imgs, status, bad


def normalize(x: np.ndarray, mean, std) -> np.ndarray:
    """fp64 definition y = (x/255 - mean_c)/std_c over a [3, H, W] (or [n,3,H,W]) uint8 array."""
    x = np.ascontiguousarray(x, np.uint8)
    mean = np.ascontiguousarray(mean, np.float64)
    std = np.ascontiguousarray(std, np.float64)
    if x.ndim == 4:
        return np.stack([normalize(xi, mean, std) for xi in x])
    y = np.zeros(x.shape, np.float64)
    lib().l3ref_normalize(x.ctypes.data, x[0].size, x.shape[0], mean.ctypes.data, std.ctypes.data, y.ctypes.data)
    return y
