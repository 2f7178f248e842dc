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

# a file cut inside a unit's data as the LAST file of an exactly-sized source
# buffer (its later offsets point past the data): CORRUPT_HEADER, and no read past the buffer
# (the sanitizer test runs with PYTORCH_NO_CUDA_MEMORY_CACHING=1: every tensor is its own allocation)
import struct  # noqa: E402


def cut_inside_unit(f, u):
    W, H, N = struct.unpack("<IIB", f[4:13])
    P = (-(-W // N)) * (-(-H // N))
    uo = np.frombuffer(f[13:13 + 12 * P], "<u4")
    return f[:13 + 12 * P + (int(uo[u]) + int(uo[u + 1])) // 2 + 1]


for N in (32, 64, 128, 200):
    tf = cut_inside_unit(l3ref.encode(imgs[1], N=N), 1)
    ts, to = pack_files([files[0], tf])
    assert ts.numel() == int(to[-1])
    tsh = shapes[[0, 1]].contiguous()
    tsz = [imgs[0].size, imgs[1].size]
    too = torch.tensor([0, tsz[0]], dtype=torch.int64, device="cuda")
    tdec = BatchDecoder(2)
    for dtype in (torch.uint8, torch.float32):
        for wide, layout in ((False, "chw"), (True, "chw"), (False, "hwc")):
            out = torch.zeros(sum(tsz), dtype=dtype, device="cuda")
            st, b = tdec.decode(ts, to, tsh, out, out_offsets=too, wide=wide, layout=layout)
            torch.cuda.synchronize()
            assert st.tolist() == [0, 3], (N, dtype, wide, layout, st.tolist())
    cr = torch.tensor([[0, 0, imgs[0].shape[1], imgs[0].shape[2], 0], [1, 2, 50, 60, 1]], dtype=torch.int32,
                      device="cuda")
    for layout in ("chw", "hwc"):
        out = torch.zeros(sum(tsz), dtype=torch.uint8, device="cuda")
        st, b = tdec.decode(ts, to, tsh, out, out_offsets=torch.tensor([0, 3 * 70 * 133], dtype=torch.int64,
                                                                        device="cuda"), crops=cr, layout=layout)
        torch.cuda.synchronize()
        print("cut", N, layout, st.tolist())
print("truncated-last cases ok")
