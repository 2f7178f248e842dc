"""Experiment: C2 decode time with the original widths vs widths rounded to a multiple of 4 (all
stores vectorisable, no ragged patches)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import l3synth  # noqa: E402
from paper_2208_08711_b200 import BatchDecoder, encode_batch  # noqa: E402


def run(shapes, label):
    imgs = [l3synth.natural(h, w, 1000 + i, l3synth.GAIN["imagenet"]) for i, (h, w) in enumerate(shapes)]
    src, offs = encode_batch(imgs)
    sh = torch.tensor(np.array(shapes, np.int32), device="cuda")
    sizes = [3 * h * w for h, w in shapes]
    oo = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64), device="cuda")
    out = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
    dec = BatchDecoder(len(shapes))
    for _ in range(5):
        dec.decode(src, offs, sh, out, out_offsets=oo)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        dec.decode(src, offs, sh, out, out_offsets=oo)
    e1.record()
    torch.cuda.synchronize()
    print(label, round(e0.elapsed_time(e1) / 100, 4), "ms", "Mpx", sum(h * w for h, w in shapes) / 1e6)


shapes = l3synth.imagenet_shapes(256)
run(shapes, "orig")
run([(h, (w // 4) * 4) for h, w in shapes], "w%4==0")
run([(h, (w // 32) * 32) for h, w in shapes], "w%32==0")
