"""CUDA-graph capture of l3_decode_batch (two launches, PDL edge): correctness and C1 latency with
graph replay vs direct calls. Dev diagnostic (GPU)."""
import json, os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import l3synth
from paper_2208_08711_b200 import BatchDecoder, encode_batch, l3
torch.cuda.set_device(0)
im = l3synth.make_batch("c1_64x64")[0]
src, offs = encode_batch([im])
shapes = torch.tensor([[64, 64]], dtype=torch.int32, device="cuda")
out = torch.zeros((1, 3, 64, 64), dtype=torch.uint8, device="cuda")
dec = BatchDecoder(1)
s = torch.cuda.Stream()
a = dec.args(src, offs, shapes, out)
with torch.cuda.stream(s):
    for _ in range(3):
        l3.l3_decode_batch(a, s)
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    l3.l3_decode_batch(a, s)
out.zero_()
g.replay()
torch.cuda.synchronize()
ok = torch.equal(out[0].cpu(), torch.from_numpy(im)) and int(dec.status[0]) == 0
def lat(fn, n=2000):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    with torch.cuda.stream(s):
        for e in ev:
            e[0].record(s); fn(); e[1].record(s)
    s.synchronize()
    us = np.array([x.elapsed_time(y) * 1e3 for x, y in ev])
    return round(float(np.median(us)), 2)
def thr(fn, n=2000):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(n): fn()
        e1.record(s)
    s.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / n, 2)
print(json.dumps({"graph_ok": ok, "direct_us_p50": lat(lambda: l3.l3_decode_batch(a, s)), "graph_us_p50": lat(g.replay),
                  "direct_us_per_call_backtoback": thr(lambda: l3.l3_decode_batch(a, s)), "graph_us_per_replay_backtoback": thr(g.replay)}))
