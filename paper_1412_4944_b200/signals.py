"""Synthetic signal workloads (the reference's benchmark input generator).

The reference benchmarks SBO on random 8x8 / 16x16 patches of a procedurally
generated scene (data.py:261-304 ``synthetic_test_image`` and data.py:182-208
``extract_patches``).  This module regenerates the same bytes with the same
numpy random streams, so a workload is named by (height, width, scene seed,
patch edge, count, patch seed) instead of being shipped.  It also provides the
Gaussian chunked workload of SURVEY.md §8(d).

Output layout is the device layout: a C-contiguous float32 array of shape
(m, p) — signal j is the contiguous row ``Y[j]`` (the reference's Fortran p x m
matrix, transposed view).  ``unit-range`` values are k/255 rounded to float32.
"""
from __future__ import annotations

import numpy as np


def scene(height: int = 512, width: int = 512, seed: int = 0) -> np.ndarray:
    """Textured 8-bit grayscale scene; same draws, in the same order, as data.py:261-304."""
    g = np.random.default_rng(seed)
    rows, cols = np.mgrid[0:height, 0:width].astype(np.float64)
    v, u = rows / height, cols / width
    img = 0.45 + 0.25 * u + 0.15 * np.sin(2.3 * np.pi * v)
    for _ in range(24):  # soft blobs
        cy, cx = g.uniform(0, 1, 2)
        rad = g.uniform(0.02, 0.18)
        amp = g.uniform(-0.35, 0.35)
        img += amp * np.exp(-((v - cy) ** 2 + (u - cx) ** 2) / (2 * rad ** 2))
    for _ in range(20):  # oriented stripes, half of them localized
        fy, fx = g.uniform(4, 150, 2)
        ph = g.uniform(0, 2 * np.pi)
        amp = g.uniform(0.01, 0.05)
        wave = np.sin(2 * np.pi * (fy * v + fx * u) + ph)
        if g.random() < 0.5:
            cy, cx = g.uniform(0, 1, 2)
            spread = g.uniform(0.05, 0.3)
            wave = wave * np.exp(-((v - cy) ** 2 + (u - cx) ** 2) / (2 * spread ** 2))
        img += amp * wave
    for _ in range(6):  # hard edges
        cut = g.uniform(0.2, 0.8)
        amp = g.uniform(-0.15, 0.15)
        img += amp * ((u > cut) if g.random() < 0.5 else (v > cut))
    img += 0.07 * g.standard_normal(img.shape)
    lo, hi = img.min(), img.max()
    img = (img - lo) / (hi - lo)
    return np.floor(img * 255.0 + 0.5).astype(np.uint8)


def patch_bytes(grid: np.ndarray, edge: int, count: int, seed: int, lo: int = 0,
                hi: int | None = None) -> np.ndarray:
    """Random edge x edge patches as uint8 rows: patches [lo, hi) of ``count``.

    Corner draws follow data.py:182-208: rows then columns from
    ``default_rng(seed).integers`` over all ``count`` patches (so a shard
    [lo, hi) gets the same bytes as the whole workload's rows lo..hi-1); each
    patch is vectorized column-major (pixel (r, c) lands at c*edge + r)."""
    grid = np.asarray(grid)
    h, w = grid.shape
    if h < edge or w < edge:
        raise ValueError(f"grid {h}x{w} is smaller than a {edge}x{edge} patch")
    hi = count if hi is None else hi
    g = np.random.default_rng(seed)
    r0 = g.integers(0, h - edge + 1, size=count)[lo:hi]
    c0 = g.integers(0, w - edge + 1, size=count)[lo:hi]
    win = np.lib.stride_tricks.sliding_window_view(grid, (edge, edge))
    n = hi - lo
    out = np.empty((n, edge * edge), np.uint8)
    step = 1 << 20
    for s in range(0, n, step):  # bounded temporaries for 16M-patch workloads
        e = min(s + step, n)
        out[s:e] = win[r0[s:e], c0[s:e]].transpose(0, 2, 1).reshape(e - s, edge * edge)
    return out


def unit_range(u8: np.ndarray) -> np.ndarray:
    """uint8 patch rows -> float32 signals k/255 (the ``unit-range`` normalization)."""
    # the 256 possible values k/255 (float64, rounded to float32) by table lookup
    return _UNIT_TABLE[np.asarray(u8, dtype=np.uint8)]


_UNIT_TABLE = (np.arange(256, dtype=np.float64) / 255.0).astype(np.float32)


def patch_signals(m: int, edge: int = 8, height: int = 512, width: int = 512,
                  scene_seed: int = 0, patch_seed: int = 11) -> np.ndarray:
    """(m, edge^2) float32 signal rows from the synthetic scene."""
    return unit_range(patch_bytes(scene(height, width, scene_seed), edge, m, patch_seed))


def gaussian_signals(p: int, m: int, seed: int = 0, chunk: int = 1 << 20) -> np.ndarray:
    """(m, p) float32 Gaussian rows in independently seeded 2^20-signal chunks.

    Chunk c draws ``default_rng(SeedSequence([seed, c])).standard_normal((p, n))``
    so any shard can regenerate its own range."""
    out = np.empty((m, p), np.float32)
    for c, s in enumerate(range(0, m, chunk)):
        n = min(chunk, m - s)
        g = np.random.default_rng(np.random.SeedSequence([seed, c]))
        out[s:s + n] = g.standard_normal((p, n)).T
    return out
