"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO persistence arithmetic: it only draws images.  Both the
oracle (``oracle/``) and the CUDA path receive the bytes produced here; neither
imports the other.

Recipes follow SURVEY.md §8(d.2) and BASELINE.json ``configs`` (BJ:7-11).  The
paper's own datasets (Lena, Bonsai, Head Aneurism, Reduced MNIST; PAPER.md:184-190,
489-496) are not available, so these seeded images stand in for them:

* C1 ``iid_uniform``   -- 2D greyscale picture in miniature.
* C2 ``random_walk``   -- the scalar time-series example at scale.
* C3 ``blobs``         -- MNIST-like 28x28 digits, 256 integer levels.
* C4 ``grf``           -- smooth CT-like volume (Bonsai/Head).
* C5 ``grf`` + ``ball_mask`` -- non-rectangular domain, +inf outside.

Every array is float32, C-order, x (the column index) is the last axis.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "iid_uniform", "random_walk", "blobs", "grf", "ball_mask", "masked_grf",
    "config", "CONFIGS", "small_int_image",
]


def iid_uniform(shape, seed: int = 1) -> np.ndarray:
    """C1: i.i.d. U[0,1) float32 pixels (BJ:7)."""
    return np.random.default_rng(seed).random(tuple(shape), dtype=np.float32)


def random_walk(n: int = 1 << 24, seed: int = 2, dtype=np.float32) -> np.ndarray:
    """C2: cumulative sum of N(0,1) steps in float64, cast to float32 (BJ:8).
    dtype=np.float64 keeps the walk in double (the float64 variant)."""
    s = np.random.default_rng(seed).standard_normal(n)
    return np.cumsum(s).astype(dtype)


def blobs(batch: int = 65536, seed: int = 3, size: int = 28, chunk: int = 4096) -> np.ndarray:
    """C3: batch of greyscale images, each a sum of 3..8 Gaussian blobs plus U[0,20) noise,
    rounded half-to-even and clipped to [0,255] (BJ:9).  Shape (batch, size, size).

    Draw order (fixed): k, cx, cy, amplitude, sigma (each (batch, 8)), then noise.
    """
    rng = np.random.default_rng(seed)
    k = rng.integers(3, 9, size=batch)
    cx = rng.uniform(0.0, size, size=(batch, 8))
    cy = rng.uniform(0.0, size, size=(batch, 8))
    amp = rng.uniform(60.0, 255.0, size=(batch, 8))
    sig = rng.uniform(1.5, 4.0, size=(batch, 8))
    noise = rng.uniform(0.0, 20.0, size=(batch, size, size))
    out = np.empty((batch, size, size), dtype=np.float32)
    yy, xx = np.meshgrid(np.arange(size, dtype=np.float64), np.arange(size, dtype=np.float64),
                         indexing="ij")
    active = (np.arange(8)[None, :] < k[:, None]).astype(np.float64)
    for s0 in range(0, batch, chunk):
        s1 = min(batch, s0 + chunk)
        dx = xx[None, None] - cx[s0:s1, :, None, None]
        dy = yy[None, None] - cy[s0:s1, :, None, None]
        r2 = dx * dx + dy * dy
        g = (amp[s0:s1] * active[s0:s1])[:, :, None, None] * np.exp(
            -r2 / (2.0 * sig[s0:s1, :, None, None] ** 2))
        img = g.sum(axis=1) + noise[s0:s1]
        out[s0:s1] = np.rint(np.clip(img, 0.0, 255.0)).astype(np.float32)
    return out


def grf(shape, sigma: float, seed: int | np.random.Generator) -> np.ndarray:
    """C4/C5: white noise N(0,1) smoothed by an isotropic Gaussian of std ``sigma`` voxels,
    applied as a periodic FFT filter exp(-2 pi^2 sigma^2 |f|^2); float64 -> float32 (BJ:10-11)."""
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    shape = tuple(int(s) for s in shape)
    w = rng.standard_normal(shape)
    freqs = [np.fft.fftfreq(n) for n in shape[:-1]] + [np.fft.rfftfreq(shape[-1])]
    grids = np.meshgrid(*freqs, indexing="ij", sparse=True)
    f2 = sum(g * g for g in grids)
    filt = np.exp(-2.0 * np.pi ** 2 * sigma ** 2 * f2)
    axes = list(range(len(shape)))
    out = np.fft.irfftn(np.fft.rfftn(w, axes=axes) * filt, s=shape, axes=axes)
    return out.astype(np.float32)


def ball_mask(shape, radius: float) -> np.ndarray:
    """True inside the closed ball of ``radius`` centred at ((n-1)/2, ...)."""
    idx = np.meshgrid(*[np.arange(n, dtype=np.float64) - (n - 1) / 2.0 for n in shape],
                      indexing="ij", sparse=True)
    r2 = sum(g * g for g in idx)
    return r2 <= radius * radius


def masked_grf(shape, sigma: float, radius: float, seed) -> np.ndarray:
    """C5: GRF with voxels outside the centred ball set to +inf."""
    v = grf(shape, sigma, seed)
    v[~ball_mask(shape, radius)] = np.inf
    return v


def small_int_image(shape, levels: int, seed: int, inf_frac: float = 0.0) -> np.ndarray:
    """Tiny fuzz images with integer levels 0..levels-1,
    optionally with random +inf voxels (non-rectangular domains, reading R5)."""
    rng = np.random.default_rng(seed)
    img = rng.integers(0, levels, size=tuple(shape)).astype(np.float32)
    if inf_frac > 0:
        img[rng.random(tuple(shape)) < inf_frac] = np.inf
    return img


# name -> (builder, description, maxdim)
CONFIGS = {
    "c1": (lambda: iid_uniform((128, 128), 1), "2D 128x128 iid U[0,1), H0+H1", 1),
    "c2": (lambda: random_walk(1 << 24, 2), "1D random walk 2^24, H0", 0),
    "c3": (lambda: blobs(65536, 3), "65536 x 28x28 blob images, H0+H1", 1),
    "c4": (lambda: grf((128, 128, 128), 2.0, 4), "3D 128^3 GRF sigma=2, H0-H2", 2),
    "c5": (lambda: masked_grf((384, 384, 384), 3.0, 180.0, 5), "3D 384^3 GRF sigma=3 in ball r=180, H0-H2", 2),
    "c5b": (lambda: np.stack([masked_grf((128, 128, 128), 3.0, 60.0, g)
                              for g in [np.random.default_rng(6)] * 64]),
            "64 x 128^3 GRF sigma=3 in ball r=60, H0-H2", 2),
}


def config(name: str):
    """Return (image, maxdim) for a BASELINE.json config name."""
    build, _, maxdim = CONFIGS[name]
    return build(), maxdim
