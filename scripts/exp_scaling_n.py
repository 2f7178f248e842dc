"""Decode time vs batch size on C3-shaped images (fp32 out): fixed overhead and tail of the persistent
launch. Dev diagnostic (GPU)."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import l3synth
from paper_2208_08711_b200 import BatchDecoder, encode_batch, l3, normalize_constants
from paper_2208_08711_b200.api import IMAGENET_MEAN, IMAGENET_STD

def main():
    torch.cuda.set_device(0)
    out_kind = sys.argv[1] if len(sys.argv) > 1 else "f32"
    imgs = l3synth.make_batch("c3_cityscapes")
    src1, offs1 = encode_batch(imgs)
    files = [src1[int(offs1[i]):int(offs1[i + 1])].cpu() for i in range(len(imgs))]
    stream = torch.cuda.Stream()
    scale, bias = normalize_constants(IMAGENET_MEAN, IMAGENET_STD)
    res = {}
    for n in (1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128):
        sel = [files[i % 32] for i in range(n)]
        offs = np.zeros(n + 1, np.int64); offs[1:] = np.cumsum([len(f) for f in sel])
        src = torch.cat(sel).cuda()
        offs_t = torch.from_numpy(offs).cuda()
        shapes = torch.tensor([[1024, 2048]] * n, dtype=torch.int32, device="cuda")
        dt = torch.float32 if out_kind == "f32" else torch.uint8
        out = torch.empty((n, 3, 1024, 2048), dtype=dt, device="cuda")
        dec = BatchDecoder(n)
        a = dec.args(src, offs_t, shapes, out, scale=scale, bias=bias, wide=os.environ.get('WIDE') == '1')
        for _ in range(3):
            l3.l3_decode_batch(a, stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for e in ev:
            e[0].record(stream); l3.l3_decode_batch(a, stream); e[1].record(stream)
        stream.synchronize()
        us = float(np.median([x.elapsed_time(y) * 1e3 for x, y in ev]))
        assert bool((dec.status[:n] == 0).all())
        res[n] = {"us": round(us, 1), "us_per_img": round(us / n, 2)}
        del out, src
        torch.cuda.empty_cache()
    print(json.dumps(res))

main()
