import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import l3synth
from oracle import l3ref
from paper_2208_08711_b200 import BatchDecoder, pack_files
from paper_2208_08711_b200.api import PipelinedLoader
imgs = [l3synth.natural(200, 300, s, 2.0) for s in range(6)]
files = [l3ref.encode(im) for im in imgs]
bad = bytearray(files[4]); bad[13 + 12 * 70 + 40] &= 0x0F
for variant in ("loader", "direct", "loader_nobad"):
    files_b = [files[:3], [files[3], bytes(bad) if variant != "loader_nobad" else files[4], files[5]]]
    outs = []
    if variant.startswith("loader"):
        loader = PipelinedLoader(3, max(sum(map(len, b)) for b in files_b), depth=2)
        hs = torch.full((4, 3), -1, dtype=torch.int32).pin_memory()
        for k, b in enumerate(files_b + files_b):
            offs = torch.tensor(np.cumsum([0] + [len(f) for f in b]), dtype=torch.int64, device="cuda")
            host = torch.from_numpy(np.frombuffer(b"".join(b), np.uint8).copy()).pin_memory()
            sh = torch.tensor([[200, 300]] * len(b), dtype=torch.int32, device="cuda")
            out = torch.full((len(b), 3, 200, 300), 7, dtype=torch.uint8, device="cuda")
            loader.submit(host, offs, sh, out, host_status=hs[k])
            outs.append(out)
        torch.cuda.synchronize()
        print(variant, hs.tolist())
    else:
        dec = BatchDecoder(3)
        for k, b in enumerate(files_b + files_b):
            src, offs = pack_files(b)
            sh = torch.tensor([[200, 300]] * len(b), dtype=torch.int32, device="cuda")
            out = torch.full((len(b), 3, 200, 300), 7, dtype=torch.uint8, device="cuda")
            st, bu = dec.decode(src, offs, sh, out)
            torch.cuda.synchronize()
            print(variant, k, st.tolist(), bu.tolist())
            outs.append(out)
    for k, out in enumerate(outs):
        ref = imgs[:3] if k % 2 == 0 else imgs[3:]
        for i in range(3):
            g = out[i].cpu().numpy()
            bad_px = np.argwhere(g != ref[i])
            if len(bad_px):
                print(variant, "batch", k, "img", i, "mismatches", len(bad_px), "first", bad_px[:3].tolist(), "last", bad_px[-1].tolist())
