"""Fixed per-launch overhead of l3_decode_batch: device time vs grid cap (max_ctas), for the C1 image and the
C3 batch, next to an empty torch kernel. Dev diagnostic (GPU)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import l3synth  # noqa: E402
from paper_2208_08711_b200 import BatchDecoder, encode_batch, l3, normalize_constants  # noqa: E402
from paper_2208_08711_b200.api import IMAGENET_MEAN, IMAGENET_STD  # noqa: E402


def timeit(fn, stream, reps):
    for _ in range(5):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for e in ev:
        e[0].record(stream)
        fn()
        e[1].record(stream)
    stream.synchronize()
    us = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    return round(float(np.median(us)), 2), round(float(us.min()), 2)


def main():
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    x = torch.zeros(1, device="cuda")
    res = {"empty_torch_kernel_us": timeit(lambda: x.add_(1), stream, 200) if False else None}
    with torch.cuda.stream(stream):
        res["empty_torch_kernel_us"] = timeit(lambda: x.add_(1), stream, 200)
    for cfg, out_kind, n_rep in (("c1_64x64", "u8", 300), ("c3_cityscapes", "f32", 30)):
        imgs = l3synth.make_batch(cfg)
        src, offs = encode_batch(imgs)
        shp = np.array([im.shape[1:] for im in imgs], np.int32)
        shapes = torch.from_numpy(shp).cuda()
        dt = torch.float32 if out_kind == "f32" else torch.uint8
        out = torch.empty((len(imgs), 3, int(shp[0, 0]), int(shp[0, 1])), dtype=dt, device="cuda")
        scale, bias = normalize_constants(IMAGENET_MEAN, IMAGENET_STD) if out_kind == "f32" else ((1,) * 3, (0,) * 3)
        dec = BatchDecoder(len(imgs))
        for cap in (0, 1, 4, 16, 148, 296, 592):
            a = dec.args(src, offs, shapes, out, scale=scale, bias=bias, max_ctas=cap)
            res[f"{cfg}_max_ctas_{cap}"] = timeit(lambda: l3.l3_decode_batch(a, stream), stream, n_rep)
            assert int((dec.status == 0).all().item()) == 1
        p = dec.args(src, offs, shapes, out, scale=scale, bias=bias)
        res[f"{cfg}_parse_only"] = timeit(lambda: l3.l3_parse_batch(p, stream), stream, n_rep)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
