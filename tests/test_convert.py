"""Dataset conversion / ratio harness: host-side loading and header parsing on
CPU; GPU encode of user images byte-identical to the oracle and decodable by the hot path."""
import json
import os

import numpy as np
import pytest
import torch

import l3synth
from oracle import l3ref
from paper_2208_08711_b200 import convert


def _write_images(d):
    from PIL import Image
    imgs = {}
    a = l3synth.natural(37, 53, 1, 1.0)
    Image.fromarray(a.transpose(1, 2, 0)).save(os.path.join(d, "a.png"))
    imgs["a"] = a
    b = l3synth.uniform_image(20, 31, 2)
    Image.fromarray(b.transpose(1, 2, 0)).save(os.path.join(d, "b.ppm"))
    imgs["b"] = b
    os.makedirs(os.path.join(d, "sub"))
    c = l3synth.natural(64, 64, 3, 2.0)
    np.save(os.path.join(d, "sub", "c.npy"), c.transpose(1, 2, 0))           # [H, W, 3]
    imgs["c"] = c
    e = l3synth.uniform_image(5, 9, 4)
    np.save(os.path.join(d, "sub", "e.npy"), e)                               # [3, H, W]
    imgs["e"] = e
    with open(os.path.join(d, "notes.txt"), "w") as fh:
        fh.write("not an image")
    return imgs


def test_list_and_load(tmp_path):
    imgs = _write_images(str(tmp_path))
    files = convert.list_images([str(tmp_path)])
    assert [os.path.splitext(os.path.basename(f))[0] for f in files] == ["a", "b", "c", "e"]
    for f in files:
        stem = os.path.splitext(os.path.basename(f))[0]
        assert np.array_equal(convert.load_planar(f), imgs[stem])


def test_load_rejects_bad_arrays(tmp_path):
    p = os.path.join(tmp_path, "x.npy")
    np.save(p, np.zeros((4, 4), np.uint8))
    with pytest.raises(ValueError):
        convert.load_planar(p)
    np.save(p, np.zeros((4, 4, 3), np.float32))
    with pytest.raises(ValueError):
        convert.load_planar(p)


def test_header_shape_and_read(tmp_path):
    im = l3synth.uniform_image(21, 34, 7)
    f = l3ref.encode(im, N=16)
    assert convert.header_shape(f) == (21, 34, 16)
    assert convert.header_shape(l3ref.encode_variant(im, N=8)) == (21, 34, 8)
    p = os.path.join(tmp_path, "x.l3")
    with open(p, "wb") as fh:
        fh.write(f)
    files, shapes = convert.read_l3_files([p, p])
    assert files == [f, f] and shapes.tolist() == [[21, 34], [21, 34]]
    with pytest.raises(ValueError):
        convert.header_shape(b"PNG\x00" + bytes(20))


def test_cli_rejects_bad_patch():
    with pytest.raises(SystemExit):
        convert.main(["--patch", "300", "x.png"])


@pytest.mark.gpu
def test_convert_gpu_matches_oracle_and_decodes(tmp_path, capsys):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2208_08711_b200 import BatchDecoder, pack_files
    src_dir, out_dir = os.path.join(tmp_path, "in"), os.path.join(tmp_path, "out")
    os.makedirs(src_dir)
    imgs = _write_images(src_dir)
    assert convert.main([src_dir, "--out", out_dir, "--batch", "3"]) == 0
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    total = 0
    for stem, im in imgs.items():
        with open(os.path.join(out_dir, stem + ".l3"), "rb") as fh:
            got = fh.read()
        assert got == l3ref.encode(im)          # byte-identical to the oracle's encoder
        total += len(got)
    raw = sum(im.size for im in imgs.values())
    assert summary["images"] == 4 and summary["raw_bytes"] == raw and summary["l3_bytes"] == total
    assert abs(summary["ratio"] - total / raw) < 1e-4
    # the converted files decode on the hot path back to the source pixels
    files, shapes = convert.read_l3_files([os.path.join(out_dir, s + ".l3") for s in imgs])
    src, offs = pack_files(files)
    sizes = [3 * int(h) * int(w) for h, w in shapes]
    oo = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64), device="cuda")
    out = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
    st, _ = BatchDecoder(len(files)).decode(src, offs, torch.from_numpy(shapes).cuda(), out, out_offsets=oo)
    torch.cuda.synchronize()
    assert st.tolist() == [0] * len(files)
    flat = out.cpu().numpy()
    for o, s, im in zip(oo.cpu().numpy(), sizes, imgs.values()):
        assert np.array_equal(flat[o:o + s].reshape(im.shape), im)
