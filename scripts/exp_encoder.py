"""GPU encoder throughput on the C3 batch (raw GB/s of the l3_encode_batch call) and byte-identity with
the oracle on a sample. Dev diagnostic (GPU)."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import l3synth
from oracle import l3ref
from paper_2208_08711_b200 import encode_batch
for cfg in ("c3_cityscapes", "c2_imagenet", "c4_uhd"):
    imgs = l3synth.make_batch(cfg)
    raw = sum(im.size for im in imgs)
    ts = []
    for _ in range(3):
        t = {}
        src, offs = encode_batch(imgs, timing=t)
        ts.append(t["encode_ms"])
    o = offs.cpu().numpy()
    f0 = src[int(o[0]):int(o[1])].cpu().numpy().tobytes()
    same = f0 == l3ref.encode(imgs[0])
    print(json.dumps({"config": cfg, "images": len(imgs), "raw_mb": round(raw / 1e6, 1), "encode_ms": round(min(ts), 3),
                      "encoder_raw_gbs": round(raw / (min(ts) / 1e3) / 1e9, 2), "image0_byte_identical": same}))
