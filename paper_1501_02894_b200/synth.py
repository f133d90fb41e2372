"""Pinned seeded synthetic image generator for the BASELINE.json configs.

SURVEY.md 8(d): three random plane cosines + Gaussian blobs + i.i.d. normal
noise, ``clip(rint(128 + sum), 0, 255)``.  Draw order (numpy default_rng):
  for k in 0..2:  a~U(20,40), f~U(1,6), theta~U(0,pi), phi~U(0,2pi)
  for b in blobs: a~U(-60,60), sigma~U(8,40), (cx, cy) = uniform(0, N, 2)
  then the noise field, row-major (strip-wise draws of consecutive rows give
  the same stream, so 16384^2 is produced strip by strip).
Both the cosine and the Gaussian terms are separable, so each strip is one
small (rows x 30) @ (30 x N) float64 matrix product -- mathematically the
survey's formula, evaluated in a fixed, reproducible order.

There is no public dataset in this path; these seeded images stand in for the
paper's Lena/baboon (absent and not needed).
"""

from __future__ import annotations

import math

import numpy as np

# BASELINE.json configs -> generator parameters (SURVEY.md 8(d) seeds).
CONFIG_IMAGES = {
    "c1": dict(size=256, seed=1, noise_sigma=6.0, n_blobs=6),
    "c2": dict(size=512, seed=2, noise_sigma=6.0, n_blobs=6),
    "c4": dict(size=512, seed=4, noise_sigma=6.0, n_blobs=6),
    "c5": dict(size=16384, seed=5, noise_sigma=10.0, n_blobs=24),
}


def _factors(n: int, rng: np.random.Generator, n_blobs: int):
    """Left (per-row) and right (per-column) factors of the smooth field."""
    lefts, rights = [], []
    x = np.arange(n, dtype=np.float64)
    for _ in range(3):
        a = rng.uniform(20.0, 40.0)
        f = rng.uniform(1.0, 6.0)
        th = rng.uniform(0.0, math.pi)
        ph = rng.uniform(0.0, 2.0 * math.pi)
        kx = 2.0 * math.pi * f * math.cos(th) / n
        ky = 2.0 * math.pi * f * math.sin(th) / n
        # a*cos(kx*x + ky*y + ph) = a*cos(ky*y+ph)*cos(kx*x) - a*sin(ky*y+ph)*sin(kx*x)
        lefts.append(lambda y, a=a, ky=ky, ph=ph: a * np.cos(ky * y + ph))
        rights.append(np.cos(kx * x))
        lefts.append(lambda y, a=a, ky=ky, ph=ph: -a * np.sin(ky * y + ph))
        rights.append(np.sin(kx * x))
    for _ in range(n_blobs):
        a = rng.uniform(-60.0, 60.0)
        s = rng.uniform(8.0, 40.0)
        cx, cy = rng.uniform(0.0, n, 2)
        lefts.append(lambda y, a=a, s=s, cy=cy: a * np.exp(-((y - cy) ** 2) / (2.0 * s * s)))
        rights.append(np.exp(-((x - cx) ** 2) / (2.0 * s * s)))
    return lefts, np.stack(rights)


def synth_image(size: int, seed: int, noise_sigma: float = 6.0, n_blobs: int = 6, strip_rows: int = 1024,
                out: np.ndarray | None = None) -> np.ndarray:
    """uint8 [size, size] image of the pinned generator."""
    rng = np.random.default_rng(seed)
    lefts, right = _factors(size, rng, n_blobs)
    img = np.empty((size, size), dtype=np.uint8) if out is None else out
    for y0 in range(0, size, strip_rows):
        y1 = min(size, y0 + strip_rows)
        y = np.arange(y0, y1, dtype=np.float64)
        left = np.stack([f(y) for f in lefts], axis=1)
        acc = left @ right
        acc += rng.normal(0.0, noise_sigma, (y1 - y0, size))
        acc += 128.0
        np.rint(acc, out=acc)
        np.clip(acc, 0.0, 255.0, out=acc)
        img[y0:y1] = acc.astype(np.uint8)
    return img


def config_image(name: str) -> np.ndarray:
    return synth_image(**CONFIG_IMAGES[name])


def batch_seeds(n: int = 256, first: int = 1000) -> list[int]:
    """c3: 256 independent 512^2 images, seeds 1000..1255."""
    return list(range(first, first + n))
