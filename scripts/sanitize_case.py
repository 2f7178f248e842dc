"""Small decode cases for compute-sanitizer (memcheck / racecheck / initcheck / synccheck): every mode
(N <= 32 whole-staged, N = 33..128 streamed, wide 8-column, N > 128 generic), ragged edges,
a corrupted file, u8 and fp32; planar, HWC (tile kernel), crop + flip (CHW and HWC); the ablation
decoders (modes 0-5) on the custom- and original-Paeth formats."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import l3synth  # noqa: E402
from oracle import l3ref  # noqa: E402
from paper_2208_08711_b200 import BatchDecoder, l3, pack_files  # noqa: E402

imgs = [l3synth.uniform_image(70, 133, 1), l3synth.natural(300, 260, 2, 3.0), l3synth.natural(64, 64, 3, 1.0),
        l3synth.uniform_image(40, 300, 4)]
Ns = [32, 128, 64, 200]
files = [l3ref.encode(im, N=N) for im, N in zip(imgs, Ns)]
bad = bytearray(files[2]); bad[-5] ^= 0xF0; files.append(bytes(bad)); imgs.append(imgs[2])
files.append(files[1][:-7]); imgs.append(imgs[1])                     # truncated -> error re-walk path
kz = bytearray(files[0]); kz[13 + 12 * 15] &= 0x0F; files.append(bytes(kz)); imgs.append(imgs[0])   # k = 0
src, offs = pack_files(files)
shapes = torch.tensor([im.shape[1:] for im in imgs], dtype=torch.int32, device="cuda")
sizes = [im.size for im in imgs]
oo = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64), device="cuda")
dec = BatchDecoder(len(files))
for dtype in (torch.uint8, torch.float32):
    for wide in ((False, True) if dtype == torch.uint8 else (False,)):
        out = torch.zeros(sum(sizes), dtype=dtype, device="cuda")
        st, b = dec.decode(src, offs, shapes, out, out_offsets=oo, wide=wide)
        torch.cuda.synchronize()
        print(dtype, wide, st.tolist())

# f3: HWC tile kernel (no crops) and the crop + flip augment variants (CHW and HWC)
crops = torch.tensor([[3, 5, im.shape[1] - 3, im.shape[2] - 5, i % 2] if im.shape[1] > 3 and im.shape[2] > 5
                      else [0, 0, im.shape[1], im.shape[2], 0] for i, im in enumerate(imgs)],
                     dtype=torch.int32, device="cuda")
csz = (3 * crops[:, 2].long() * crops[:, 3].long()).cpu().numpy()
coo = torch.tensor(np.concatenate([[0], np.cumsum(csz)[:-1]]).astype(np.int64), device="cuda")
for dtype in (torch.uint8, torch.float32):
    for layout in ("hwc", "chw"):
        for cr in ((None, crops) if layout == "hwc" else (crops,)):
            out = torch.zeros(sum(sizes), dtype=dtype, device="cuda")
            st, b = dec.decode(src, offs, shapes, out, out_offsets=oo if cr is None else coo, crops=cr,
                               layout=layout)
            torch.cuda.synchronize()
            print(dtype, layout, cr is not None, st.tolist())

# f2: ablation decoders on valid files, both formats
vimgs = imgs[:4]
for files_v in ([l3ref.encode(im, N=N) for im, N in zip(vimgs, Ns)],
                [l3ref.encode_variant(im, N=N) for im, N in zip(vimgs, Ns)]):
    vs, vo = pack_files(files_v)
    vsh = shapes[:4].contiguous()
    voo = oo[:4].contiguous()
    for mode in range(6):
        out = torch.zeros(sum(sizes[:4]), dtype=torch.uint8, device="cuda")
        a = dec.args(vs, vo, vsh, out, out_offsets=voo)
        l3.l3_decode_batch_ablation(a, mode)
        torch.cuda.synchronize()
        print("ablation", mode, dec.status[:4].tolist())
