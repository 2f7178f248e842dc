"""Seeded synthetic RGB8 image generators shared by tests, smoke() and bench.py.

This module holds NO L3 arithmetic (no predictor, no base-delta, no container):
it only draws pixels. Both the oracle side (tests) and the CUDA side (bench,
parity tests) receive the same uint8 planar [3, H, W] arrays from here.

Recipes (after SURVEY.md §8(d) probe 6):

* ``gradient(H, W, seed)`` — config 1: per-channel linear gradient + U(-2, 2)
  noise.
* ``natural(H, W, seed, gain)`` — smooth field (tilt + low-frequency sinusoid)
  plus U(-1, 1) noise whose amplitude is drawn per 64×64 block from
  {0,1,2,4,8,16} with probabilities {.10,.25,.25,.20,.12,.08}, times a global
  gain calibrated so the oracle's compression ratio matches PAPER.md Table 4
  (Cityscapes 0.44, KITTI 0.64, RAISE-1K 0.63).
* ``random_image`` / ``black_image`` — Table 4's synthetic "Random" and
  "Black" rows.
* ``imagenet_shapes(n, seed)`` — ~500×375 landscape / 375×500 portrait
  (75/25), each side jittered uniformly by ±64 px.
"""
from __future__ import annotations

import numpy as np

# Calibrated global gains (scripts/calibrate_gains.py, oracle ratio).
GAIN = {"cityscapes": 0.48, "imagenet": 2.444, "uhd": 2.137}
AMPS = np.array([0, 1, 2, 4, 8, 16], dtype=np.float64)
AMP_P = np.array([0.10, 0.25, 0.25, 0.20, 0.12, 0.08])


def gradient(H: int, W: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    coef = [(1.5, 0.8, 40.0), (0.7, -1.2, 128.0), (-1.0, 1.9, 90.0)]
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    out = np.empty((3, H, W), np.uint8)
    for c, (a, b, k) in enumerate(coef):
        f = a * x + b * y + k + rng.uniform(-2.0, 2.0, size=(H, W))
        out[c] = np.clip(np.rint(f), 0, 255).astype(np.uint8)
    return out


def natural(H: int, W: int, seed: int, gain: float) -> np.ndarray:
    rng = np.random.default_rng(seed)
    y = np.arange(H, dtype=np.float64)[:, None]
    x = np.arange(W, dtype=np.float64)[None, :]
    by, bx = -(-H // 64), -(-W // 64)
    out = np.empty((3, H, W), np.uint8)
    for c in range(3):
        sx, sy = rng.uniform(-0.05, 0.05, size=2)
        lx, ly = rng.uniform(200.0, 800.0, size=2)
        phi = rng.uniform(0.0, 1.0)
        f = 128.0 + sx * x + sy * y + 40.0 * np.sin(2 * np.pi * (x / lx + phi)) * np.cos(2 * np.pi * y / ly)
        amp_blocks = AMPS[rng.choice(len(AMPS), size=(by, bx), p=AMP_P)]
        amp = np.repeat(np.repeat(amp_blocks, 64, axis=0), 64, axis=1)[:H, :W]
        f = f + rng.uniform(-1.0, 1.0, size=(H, W)) * amp * gain
        out[c] = np.clip(np.rint(f), 0, 255).astype(np.uint8)
    return out


def random_image(H: int, W: int, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, 256, size=(3, H, W), dtype=np.uint8)


def black_image(H: int, W: int) -> np.ndarray:
    return np.zeros((3, H, W), np.uint8)


def uniform_image(H: int, W: int, seed: int = 0) -> np.ndarray:
    """Arbitrary bytes with small patches of structure — for edge-case parity."""
    rng = np.random.default_rng(seed)
    kind = rng.integers(0, 3)
    if kind == 0:
        return rng.integers(0, 256, size=(3, H, W), dtype=np.uint8)
    if kind == 1:
        return natural(H, W, int(rng.integers(1 << 30)), float(rng.uniform(0.2, 4.0)))
    base = rng.integers(0, 256, size=(3, 1, 1))
    return ((base + rng.integers(-3, 4, size=(3, H, W))) % 256).astype(np.uint8)


def imagenet_shapes(n: int, seed: int = 1) -> list[tuple[int, int]]:
    """(H, W) pairs: 75% landscape ~375x500, 25% portrait ~500x375, ±64 px jitter."""
    rng = np.random.default_rng(seed)
    shapes = []
    for _ in range(n):
        landscape = rng.uniform() < 0.75
        H, W = (375, 500) if landscape else (500, 375)
        H += int(rng.integers(-64, 65))
        W += int(rng.integers(-64, 65))
        shapes.append((H, W))
    return shapes


# Workload recipes keyed by BASELINE.json config.
CONFIGS = {
    "c1_64x64": dict(n=1, shape=(64, 64), kind="gradient", seed0=0),
    "c2_imagenet": dict(n=256, shape=None, kind="natural", gain="imagenet", seed0=1000),
    "c3_cityscapes": dict(n=32, shape=(1024, 2048), kind="natural", gain="cityscapes", seed0=2000),
    "c4_uhd": dict(n=16, shape=(2160, 3840), kind="natural", gain="uhd", seed0=3000),
    # ablation-only workloads (the Fig. 10 study rescales Cityscapes to HD / FHD / UHD)
    "ab_hd": dict(n=32, shape=(720, 1280), kind="natural", gain="cityscapes", seed0=4000),
    "ab_fhd": dict(n=32, shape=(1080, 1920), kind="natural", gain="cityscapes", seed0=5000),
}


def make_batch(config: str, n: int | None = None) -> list[np.ndarray]:
    """The seeded image list of a config (optionally only its first n images)."""
    cfg = CONFIGS[config]
    count = cfg["n"] if n is None else min(n, cfg["n"])
    shapes = imagenet_shapes(cfg["n"]) if cfg["shape"] is None else [cfg["shape"]] * cfg["n"]
    imgs = []
    for i in range(count):
        H, W = shapes[i]
        if cfg["kind"] == "gradient":
            imgs.append(gradient(H, W, cfg["seed0"] + i))
        else:
            imgs.append(natural(H, W, cfg["seed0"] + i, GAIN[cfg["gain"]]))
    return imgs
