"""Measurement only (build_ab/skp.so, -DL3_DEV_SKIP_PREP): the decode-call time of C3 fp32 / u8 with and
without the a1 launch (L3_SKIP_PREP=1 reuses the previous identical call's a1 results), to bound what
folding a1 into the decode grid could gain."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2208_08711_b200 import BatchDecoder, encode_batch, l3, normalize_constants  # noqa: E402
from paper_2208_08711_b200.api import IMAGENET_MEAN, IMAGENET_STD  # noqa: E402

imgs = bench.rank_images("c3_cityscapes", 0)
src, offs = encode_batch(imgs)
shapes = torch.tensor(np.array([im.shape[1:] for im in imgs], np.int32), device="cuda")
n = len(imgs)
dec = BatchDecoder(n)
s = torch.cuda.Stream()
for out_kind in ("f32", "u8"):
    dt = torch.float32 if out_kind == "f32" else torch.uint8
    out = torch.empty((n, 3, 1024, 2048), dtype=dt, device="cuda")
    sc, bi = normalize_constants(IMAGENET_MEAN, IMAGENET_STD) if out_kind == "f32" else ((1, 1, 1), (0, 0, 0))
    a = dec.args(src, offs, shapes, out, scale=sc, bias=bi)
    for _ in range(10):
        l3.l3_decode_batch(a, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(200):
        l3.l3_decode_batch(a, s)
    e1.record(s)
    e1.synchronize()
    assert bool((dec.status[:n] == 0).all())
    print(out_kind, "skip_prep" if os.environ.get("L3_SKIP_PREP") else "with_prep", round(e0.elapsed_time(e1) / 200, 4))
