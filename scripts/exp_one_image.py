"""Decode ONE C3 image (fp32) a few times: the latency of a lone patch per warp (dev diagnostic, for ncu)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import l3synth
from paper_2208_08711_b200 import BatchDecoder, encode_batch, l3, normalize_constants
from paper_2208_08711_b200.api import IMAGENET_MEAN, IMAGENET_STD
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
imgs = [l3synth.natural(1024, 2048, 2000 + i, l3synth.GAIN["cityscapes"]) for i in range(n)]
src, offs = encode_batch(imgs)
shapes = torch.tensor([[1024, 2048]] * n, dtype=torch.int32, device="cuda")
out = torch.empty((n, 3, 1024, 2048), dtype=torch.float32, device="cuda")
scale, bias = normalize_constants(IMAGENET_MEAN, IMAGENET_STD)
dec = BatchDecoder(n)
a = dec.args(src, offs, shapes, out, scale=scale, bias=bias, max_ctas=int(os.environ.get("MAXC", "0")))
for _ in range(5):
    l3.l3_decode_batch(a)
torch.cuda.synchronize()
print("ok", dec.status.tolist()[:n])
