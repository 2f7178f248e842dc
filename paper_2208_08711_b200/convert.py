"""Dataset conversion to L3 on the GPU, and the compression-ratio harness of SURVEY.md §8 f4.

PAPER.md:246-268 (§5.2, Table 4) reports the compression ratio (compressed size / decompressed
size, lower is better) of L3 on real datasets. Those datasets are not in this sandbox, so this tool
computes the same figure for any images a user supplies. It also converts them to ``.l3`` files for
training, which is the offline step the paper assumes.

    python -m paper_2208_08711_b200.convert IMG_OR_DIR... [--out DIR] [--batch 64] [--patch N]

Inputs: anything Pillow opens (PNG, PPM, BMP, TIFF, lossless WebP, ...), converted to RGB8. Also
``.npy`` arrays of uint8, shaped [H, W, 3] or [3, H, W]. Encoding runs in the GPU encoder
(``l3_encode_batch``), which is byte-identical to the oracle's encoder
(tests/test_gpu_parity.py::test_gpu_encoder_*). Prints one JSON summary line.

Reading back: :func:`read_l3_files` returns the files and their (H, W) from the headers.
That is the host-side input of :class:`~paper_2208_08711_b200.BatchDecoder` /
:class:`~paper_2208_08711_b200.api.PipelinedLoader`.
"""
from __future__ import annotations

import argparse
import json
import os
import struct
import sys
from typing import Iterable, Sequence

import numpy as np

IMAGE_EXT = {".png", ".ppm", ".pnm", ".bmp", ".tif", ".tiff", ".webp", ".npy", ".jpg", ".jpeg"}


def list_images(paths: Sequence[str]) -> list[str]:
    """Files given directly, plus the image files under any directory (sorted, recursive)."""
    out: list[str] = []
    for p in paths:
        if os.path.isdir(p):
            for root, _dirs, files in os.walk(p):
                out.extend(os.path.join(root, f) for f in sorted(files) if os.path.splitext(f)[1].lower() in IMAGE_EXT)
        else:
            out.append(p)
    return sorted(out)


def load_planar(path: str) -> np.ndarray:
    """uint8 planar [3, H, W] (R, G, B) from an image file or a .npy array."""
    if path.lower().endswith(".npy"):
        a = np.load(path)
        if a.dtype != np.uint8 or a.ndim != 3:
            raise ValueError(f"{path}: expected a uint8 [H, W, 3] or [3, H, W] array, got {a.dtype} {a.shape}")
        if a.shape[0] == 3 and a.shape[2] != 3:
            return np.ascontiguousarray(a)
        if a.shape[2] == 3:
            return np.ascontiguousarray(a.transpose(2, 0, 1))
        raise ValueError(f"{path}: no channel axis of size 3 in {a.shape}")
    from PIL import Image
    with Image.open(path) as im:
        rgb = np.asarray(im.convert("RGB"), dtype=np.uint8)
    return np.ascontiguousarray(rgb.transpose(2, 0, 1))


def header_shape(f: bytes) -> tuple[int, int, int]:
    """(H, W, N) from an L3 header (reading C9: "L3IF" | W u32le | H u32le | N u8)."""
    if len(f) < 13 or f[:4] not in (b"L3IF", b"L3IP"):
        raise ValueError("not an L3 file")
    W, H, N = struct.unpack("<IIB", f[4:13])
    return H, W, N


def read_l3_files(paths: Iterable[str]) -> tuple[list[bytes], np.ndarray]:
    """The files' bytes and an int32 [n, 2] array of their (H, W)."""
    files = []
    for p in paths:
        with open(p, "rb") as fh:
            files.append(fh.read())
    shapes = np.array([header_shape(f)[:2] for f in files], np.int32).reshape(len(files), 2)
    return files, shapes


def convert(paths: Sequence[str], out_dir: str | None = None, batch: int = 64, patch: int = 0,
            predictor: int = 0, device: str = "cuda") -> dict:
    """Encode every image on the GPU; optionally write <out_dir>/<stem>.l3. Returns the summary."""
    from .api import encode_batch
    files = list_images(paths)
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
    raw = comp = 0
    ratios = []
    enc_ms = 0.0
    for b0 in range(0, len(files), batch):
        chunk = files[b0:b0 + batch]
        imgs = [load_planar(p) for p in chunk]
        timing = {}
        src, offs = encode_batch(imgs, patch_sizes=[patch] * len(imgs), device=device, predictor=predictor,
                                 timing=timing)
        enc_ms += timing["encode_ms"]
        o = offs.cpu().numpy()
        buf = src.cpu().numpy() if int(o[-1]) else np.zeros(0, np.uint8)
        for p, im, a, b in zip(chunk, imgs, o[:-1], o[1:]):
            nbytes = int(b - a)
            raw += im.size
            comp += nbytes
            ratios.append(nbytes / im.size)
            if out_dir:
                stem = os.path.splitext(os.path.basename(p))[0]
                with open(os.path.join(out_dir, stem + ".l3"), "wb") as fh:
                    fh.write(buf[int(a):int(b)].tobytes())
        del src, offs
    return {
        "images": len(files),
        "raw_bytes": raw,
        "l3_bytes": comp,
        "ratio": round(comp / raw, 4) if raw else None,   # Table 4's figure: compressed / decompressed
        "ratio_min": round(min(ratios), 4) if ratios else None,
        "ratio_max": round(max(ratios), 4) if ratios else None,
        "format": "L3IP (original Paeth)" if predictor else "L3IF",
        "patch": patch or "policy (PAPER.md:166)",
        # the GPU encoder alone (l3_encode_batch device time, images already in HBM): raw input bytes / s
        "encode_ms": round(enc_ms, 3),
        "encoder_raw_gbs": round(raw / (enc_ms / 1e3) / 1e9, 2) if enc_ms > 0 else None,
    }


def main(argv: Sequence[str] | None = None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("inputs", nargs="+", help="image files and / or directories")
    ap.add_argument("--out", default=None, help="write <stem>.l3 files here")
    ap.add_argument("--batch", type=int, default=64, help="images per GPU encode call")
    ap.add_argument("--patch", type=int, default=0, help="patch size N (0 = the paper's policy)")
    ap.add_argument("--original-paeth", action="store_true", help="write the ablation variant L3IP (reading C16)")
    a = ap.parse_args(argv)
    if not 0 <= a.patch <= 255:
        ap.error("--patch must be in 0..255")
    summary = convert(a.inputs, a.out, a.batch, a.patch, 1 if a.original_paeth else 0)
    print(json.dumps(summary), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
