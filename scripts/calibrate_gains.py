"""Bisect l3synth's global noise gain so the ORACLE's compression ratio on the
config's first images matches PAPER.md Table 4 (:259): Cityscapes 0.44 (C3),
KITTI 0.64 (C2, the N=32 regime), RAISE-1K 0.63 (C4). Calls only oracle/ and
l3synth; prints the gains to paste into l3synth.GAIN."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import l3synth  # noqa: E402
from oracle import l3ref  # noqa: E402

TARGET = {"c3_cityscapes": ("cityscapes", 0.44, 3), "c2_imagenet": ("imagenet", 0.64, 32),
          "c4_uhd": ("uhd", 0.63, 2)}


def ratio(cfg, gain, count):
    l3synth.GAIN[TARGET[cfg][0]] = gain
    imgs = l3synth.make_batch(cfg, count)
    return sum(len(l3ref.encode(im)) for im in imgs) / sum(im.size for im in imgs)


for cfg, (key, tgt, count) in TARGET.items():
    lo, hi = 0.05, 8.0
    for _ in range(14):
        mid = 0.5 * (lo + hi)
        if ratio(cfg, mid, count) < tgt:
            lo = mid
        else:
            hi = mid
    g = round(0.5 * (lo + hi), 3)
    print(cfg, key, g, round(ratio(cfg, g, count), 4))
