"""User-facing wrappers over the C ABI: buffer management, no arithmetic.

* :class:`BatchDecoder` — owns the device workspace / status buffers of one
  stream and decodes a batch of L3 files resident in HBM into a u8 or fp32
  ``[n, 3, H, W]`` tensor (or per-image blocks of a flat tensor for mixed
  shapes) with one ``l3_decode_batch`` call.
* :func:`encode_batch` — converts planar uint8 images to L3 files with the GPU
  encoder (``l3_encode_batch``), returning the concatenated files on device.
* :func:`normalize_constants` — host-side float32 (scale, bias) with
  ``y = fmaf(x, scale, bias) == (x/255 - mean)/std`` up to rounding.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import l3

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def wide_hint(shapes_hw, out_dtype) -> bool:
    """The L3_DECODE_HINT_WIDE choice for a batch (a performance hint only; u8 output): most images
    get a patch size N > 32 from the encoder's policy (asked of the library through
    l3_choose_patch_size) and the batch has enough patches (>= 16k units, e.g. 16 x UHD) that
    2-patch tasks still keep every warp busy (measured: wins on config 4, loses on 32 x 2048x1024;
    DESIGN.md §5)."""
    if out_dtype != torch.uint8 or len(shapes_hw) == 0:
        return False
    big = 0
    units = 0
    for h, w in shapes_hw:
        h, w = int(h), int(w)
        n = l3.l3_choose_patch_size(w, h)
        units += 3 * (-(-h // n)) * (-(-w // n))
        big += n > 32
    return 2 * big >= len(shapes_hw) and units >= 16384


def normalize_constants(mean: Sequence[float], std: Sequence[float]):
    """scale_c = 1/(255 std_c), bias_c = -mean_c/std_c, rounded once to float32."""
    scale = tuple(float(np.float32(1.0 / (255.0 * s))) for s in std)
    bias = tuple(float(np.float32(-m / s)) for m, s in zip(mean, std))
    return scale, bias


class BatchDecoder:
    """Reusable decode context (workspace + status) for batches of up to `max_n` images."""

    def __init__(self, max_n: int, device: torch.device | str = "cuda"):
        if not torch.cuda.is_available():
            raise RuntimeError("BatchDecoder needs a CUDA device (the decoder has no CPU path)")
        self.device = torch.device(device)
        self.max_n = max_n
        ws = l3.l3_decode_workspace_size(max_n)
        self.workspace = torch.zeros(ws, dtype=torch.uint8, device=self.device)   # zero before first use
        self.status = torch.empty(max_n, dtype=torch.int32, device=self.device)
        self.bad_unit = torch.empty(max_n, dtype=torch.int32, device=self.device)

    def args(self, src, src_offsets, shapes, out, *, out_offsets=None, scale=(1.0, 1.0, 1.0),
             bias=(0.0, 0.0, 0.0), wide=False, crops=None, layout="chw", max_ctas=0):
        n = int(shapes.shape[0])
        if layout not in ("chw", "hwc"):
            raise ValueError(f"layout must be 'chw' or 'hwc', got {layout!r}")
        flags = (l3.L3_DECODE_HINT_WIDE if wide else 0) | (l3.L3_DECODE_LAYOUT_HWC if layout == "hwc" else 0)
        if n > self.max_n:
            raise ValueError(f"batch of {n} > max_n={self.max_n}")
        return l3.make_decode_args(src, src_offsets, shapes, out, self.status[:n], self.workspace,
                                   out_offsets=out_offsets, bad_unit=self.bad_unit[:n], scale=scale, bias=bias,
                                   flags=flags, crops=crops, max_ctas=max_ctas)

    def decode(self, src: torch.Tensor, src_offsets: torch.Tensor, shapes: torch.Tensor,
               out: torch.Tensor, *, out_offsets=None, scale=(1.0, 1.0, 1.0), bias=(0.0, 0.0, 0.0),
               stream=None, wide=False, crops=None, layout="chw", max_ctas=0):
        """Enqueue one batch decode on `stream`; returns (status, bad_unit) device views.
        wide: performance hint for u8 batches of large images (policy N = 128), see l3.h.
        crops: optional int32 [n, 5] device tensor {y, x, h, w, flip}: decode only that window.
        layout: "chw" (planar, default) or "hwc" (interleaved, L3_DECODE_LAYOUT_HWC).
        max_ctas: cap on the decoder's thread blocks (0 = every SM), to leave SMs to compute."""
        a = self.args(src, src_offsets, shapes, out, out_offsets=out_offsets, scale=scale, bias=bias, wide=wide,
                      crops=crops, layout=layout, max_ctas=max_ctas)
        l3.l3_decode_batch(a, stream)
        n = int(shapes.shape[0])
        return self.status[:n], self.bad_unit[:n]


def pack_files(files: Sequence[bytes], device="cuda"):
    """Concatenate L3 files into one 16-byte aligned device buffer + int64 offsets (n+1)."""
    offs = np.zeros(len(files) + 1, np.int64)
    offs[1:] = np.cumsum([len(f) for f in files])
    host = np.frombuffer(b"".join(files), np.uint8) if offs[-1] else np.zeros(0, np.uint8)
    src = torch.empty(max(int(offs[-1]), 1), dtype=torch.uint8, device=device)
    if offs[-1]:
        src[: int(offs[-1])].copy_(torch.from_numpy(host.copy()))
    return src, torch.from_numpy(offs).to(device)


def encode_batch(images: Sequence[np.ndarray] | Sequence[torch.Tensor], patch_sizes=None, device="cuda",
                 stream=None, predictor: int = 0, timing: dict | None = None):
    """GPU-encode planar uint8 [3, H, W] images. Returns (src, src_offsets) on device.
    predictor=1 writes the original-Paeth ablation variant "L3IP" (reading C16).
    timing: if a dict, its "encode_ms" gets the device time of the l3_encode_batch call (CUDA events
    on its stream; the images are already in HBM)."""
    n = len(images)
    shapes = np.array([tuple(im.shape[1:]) for im in images], np.int32).reshape(n, 2)
    sizes = np.array([3 * int(h) * int(w) for h, w in shapes], np.int64)
    img_off = np.zeros(n, np.uint64)
    if n > 1:
        img_off[1:] = np.cumsum(sizes)[:-1]
    flat = torch.empty(max(int(sizes.sum()), 1), dtype=torch.uint8, device=device)
    for im, o, s in zip(images, img_off, sizes):
        t = im if isinstance(im, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(im))
        flat[int(o):int(o) + int(s)].copy_(t.reshape(-1), non_blocking=False)
    nh = None if patch_sizes is None else np.ascontiguousarray(patch_sizes, np.int32)
    cap = sum(l3.l3_encode_max_bytes(int(w), int(h), 0 if nh is None else int(nh[i]))
              for i, (h, w) in enumerate(shapes))
    dst = torch.empty(max(cap, 1), dtype=torch.uint8, device=device)
    dst_offsets = torch.empty(n + 1, dtype=torch.int64, device=device)
    ws = torch.empty(max(l3.l3_encode_workspace_size(shapes, nh), 256), dtype=torch.uint8, device=device)
    es = torch.cuda.current_stream(dst.device) if stream is None else stream
    if timing is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(es)
    l3.l3_encode_batch(flat, img_off, shapes, nh, dst, dst_offsets, ws, stream, predictor=predictor)
    if timing is not None:
        e1.record(es)
    es.synchronize()
    if timing is not None:
        timing["encode_ms"] = e0.elapsed_time(e1)
    total = int(dst_offsets[-1].item())
    src = torch.empty(max(total, 1), dtype=torch.uint8, device=device)
    src[:total].copy_(dst[:total])
    return src, dst_offsets


class PipelinedLoader:
    """Load + decode pipeline (SURVEY.md §8(f1); PAPER.md:67 Load stage, :189 "we allocate both
    processes to separate CUDA streams. We prioritize the computing stream over the decoding
    stream"). Every batch goes through ONE C-ABI call with host buffers, l3_load_decode_batch:
    pinned host bytes -> HBM, the decode kernel, statuses -> pinned host, all on one stream.
    Consecutive batches alternate over `depth` streams, each with its own device staging buffer
    and workspace, so batch i+1's host-to-device copy overlaps batch i's decode. The streams get
    the LOWEST priority, so a training step on a high-priority compute stream is scheduled first;
    `max_ctas` can further cap the decoder's thread blocks (l3.h) to leave SMs to compute.

    submit() enqueues one batch and returns a ticket; wait(ticket) blocks until that batch is
    done and returns its host statuses. The loader holds references to a batch's host and device
    buffers until its slot is reused (the asynchronous copies are invisible to torch's allocators);
    a submit that reuses a slot first waits for the slot's previous batch. With the internal status buffers a ticket must be waited
    for before `depth` more batches are submitted (its slot is then reused; wait raises); pass
    host_status= (pinned, >= n int32) to keep every batch's statuses."""

    def __init__(self, max_n: int, max_bytes: int, depth: int = 2, device="cuda", max_ctas: int = 0):
        lowest, _highest = torch.cuda.Stream.priority_range()
        self.device = torch.device(device)
        self.depth = depth
        self.max_ctas = max_ctas
        self.streams = [torch.cuda.Stream(device=self.device, priority=lowest) for _ in range(depth)]
        self.stage = [torch.empty(max_bytes + 16, dtype=torch.uint8, device=self.device) for _ in range(depth)]
        self.dec = [BatchDecoder(max_n, self.device) for _ in range(depth)]
        self.host_status = [torch.empty(max_n, dtype=torch.int32).pin_memory() for _ in range(depth)]
        self.done = [torch.cuda.Event() for _ in range(depth)]
        self.owner = [-1] * depth
        self.keep = [None] * depth      # host buffers of the batch in flight on each slot
        self.i = 0

    def submit(self, host_src: torch.Tensor, src_offsets: torch.Tensor, shapes: torch.Tensor, out: torch.Tensor,
               *, out_offsets=None, scale=(1.0, 1.0, 1.0), bias=(0.0, 0.0, 0.0), wide=False,
               host_status: torch.Tensor | None = None) -> int:
        b = self.i % self.depth
        n = int(shapes.shape[0])
        if host_src.numel() > self.stage[b].numel():
            raise ValueError("batch larger than the loader's staging buffers")
        hs = self.host_status[b] if host_status is None else host_status
        if self.keep[b] is not None:
            # the slot's previous batch must be done before its staging buffer, workspace and host
            # buffers are reused (the copies run asynchronously, outside torch's pinned-memory tracking)
            self.done[b].synchronize()
        a = self.dec[b].args(self.stage[b], src_offsets, shapes, out, out_offsets=out_offsets, scale=scale,
                             bias=bias, wide=wide, max_ctas=self.max_ctas)
        # the caller's device tensors (offsets, shapes, out) were produced on its current stream: the
        # loader's non-blocking stream must not run ahead of that work
        self.streams[b].wait_stream(torch.cuda.current_stream(self.device))
        l3.l3_load_decode_batch(a, host_src, hs[:n], self.streams[b])
        self.done[b].record(self.streams[b])
        self.keep[b] = (host_src, hs, src_offsets, shapes, out, out_offsets)
        self.owner[b] = self.i
        self.i += 1
        return self.i - 1

    def wait(self, ticket: int) -> torch.Tensor:
        """Block until batch `ticket` is decoded; returns the internal host status buffer of its slot
        (only meaningful if the batch was submitted without host_status=)."""
        b = ticket % self.depth
        if self.owner[b] != ticket:
            raise RuntimeError(f"ticket {ticket}: its slot was reused by ticket {self.owner[b]}; wait earlier "
                               f"or pass host_status= to submit")
        self.done[b].synchronize()
        return self.host_status[b]
