"""C2 (ImageNet-shaped, N = 32) decode time: planar vs HWC (tile kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import l3synth  # noqa: E402
from paper_2208_08711_b200 import BatchDecoder, encode_batch  # noqa: E402

shapes = l3synth.imagenet_shapes(256)
imgs = [l3synth.natural(h, w, 1000 + i, l3synth.GAIN["imagenet"]) for i, (h, w) in enumerate(shapes)]
src, offs = encode_batch(imgs)
sh = torch.tensor(np.array(shapes, np.int32), device="cuda")
sizes = [3 * h * w for h, w in shapes]
oo = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64), device="cuda")
dec = BatchDecoder(len(shapes))
for dt in (torch.uint8, torch.float32):
    out = torch.empty(sum(sizes), dtype=dt, device="cuda")
    for layout in ("chw", "hwc"):
        for _ in range(5):
            dec.decode(src, offs, sh, out, out_offsets=oo, layout=layout)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            dec.decode(src, offs, sh, out, out_offsets=oo, layout=layout)
        e1.record()
        torch.cuda.synchronize()
        assert bool((dec.status[:256] == 0).all())
        print(dt, layout, round(e0.elapsed_time(e1) / 50, 4), "ms")
