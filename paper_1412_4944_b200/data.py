"""Signal ingestion on the device — SURVEY.md 8(f) row 3 (data.py:182-208, 261-304).

``extract_patches(grid, cfg)`` is the reference's function (same arguments,
validation messages and result: a Fortran-ordered float64 (edge^2, count)
matrix, bit-identical) with the gather, the /255 scaling and the optional patch
mean removal done by ``sbo_extract_patches`` on the GPU.  The corner draws stay
in numpy (``default_rng(seed).integers``, rows then columns), so the sampled
positions are the reference's exactly.

``extract_patches_device`` stops before the host: it returns the signals as
device rows (an ``engine.Signals``), which ``sbo_train`` / ``represent`` accept
in place of a host matrix — a workload then crosses PCIe as the 8-bit grid plus
the corner indices instead of the float signal matrix.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .engine import Signals, require_device
from .signals import scene as synthetic_test_image  # data.py:261-304, same bytes

NORMALIZATIONS = ("unit-range", "unit-range-dc-removed")
GRID_U8, GRID_F64 = 0, 1


@dataclass
class PatchConfig:
    """data.py:37-54 — random square-patch extraction settings."""

    patch_edge: int = 8
    count: int = 4096
    seed: int = 0
    normalization: str = "unit-range"

    def validate(self) -> None:
        if self.patch_edge < 1:
            raise ValueError(f"patch_edge must be at least 1, got {self.patch_edge}")
        if self.count < 1:
            raise ValueError(f"count must be at least 1, got {self.count}")
        if self.normalization not in NORMALIZATIONS:
            raise ValueError(
                f"normalization must be one of {NORMALIZATIONS}, got {self.normalization!r}"
            )


def _check_grid(grid, e: int) -> np.ndarray:
    grid = np.asarray(grid)
    if grid.ndim != 2:
        raise ValueError(f"expected a 2-D grayscale grid, got shape {grid.shape}")
    h, w = grid.shape
    if h < e or w < e:
        raise ValueError(f"grid {h}x{w} is smaller than a {e}x{e} patch")
    return grid


def patch_corners(h: int, w: int, edge: int, count: int, seed: int):
    """data.py:199-201 — top-left corners, uniform with replacement (rows, then cols)."""
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, h - edge + 1, size=count)
    cols = rng.integers(0, w - edge + 1, size=count)
    return rows, cols


def upload_grid(grid: np.ndarray, device) -> tuple[torch.Tensor, int]:
    """The grid on the device as uint8 when it is 8-bit, else float64 (every other
    numeric dtype converts to float64 exactly as the reference's astype does)."""
    if grid.dtype == np.uint8:
        return torch.from_numpy(np.ascontiguousarray(grid)).to(device), GRID_U8
    g = np.ascontiguousarray(grid, dtype=np.float64)
    return torch.from_numpy(g).to(device), GRID_F64


def extract_rows(grid_dev: torch.Tensor, grid_code: int, edge: int, rows_dev: torch.Tensor,
                 cols_dev: torch.Tensor, normalization: str, dtype=torch.float64,
                 out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Device form: (count, edge^2) signal rows from a device grid and device int32
    corners (stream-ordered on the current stream unless ``stream`` is given)."""
    if normalization not in NORMALIZATIONS:
        raise ValueError(f"normalization must be one of {NORMALIZATIONS}, got {normalization!r}")
    if dtype == torch.float32 and normalization != "unit-range":
        raise ValueError("float32 rows are only offered for the unit-range normalization")
    h, w = grid_dev.shape
    count = rows_dev.numel()
    if out is None:
        out = torch.empty((count, edge * edge), dtype=dtype, device=grid_dev.device)
    st = torch.cuda.current_stream(grid_dev.device).cuda_stream if stream is None else stream
    L.call("sbo_extract_patches", grid_dev.data_ptr(), grid_code, h, w, grid_dev.stride(0), edge,
           rows_dev.data_ptr(), cols_dev.data_ptr(), count, NORMALIZATIONS.index(normalization),
           L.F32 if out.dtype == torch.float32 else L.F64, out.data_ptr(), st)
    return out


def extract_patches_device(grid, cfg: PatchConfig, device=None, dtype=torch.float64) -> Signals:
    """Patches as device signal rows (``Signals``).  float64 rows are the reference's
    values bit for bit; float32 rows (unit-range only) are their round-to-nearest —
    the benchmark's float32 signals."""
    cfg.validate()
    e = cfg.patch_edge
    grid = _check_grid(grid, e)
    if e * e > 1024:
        raise ValueError(f"patch_edge {e} exceeds the device ingestion limit of 32")
    dev = require_device(None if device is None else torch.device(device).index)
    h, w = grid.shape
    if max(h, w) >= 2 ** 31:
        raise ValueError("grid dimensions must be below 2^31")
    rows, cols = patch_corners(h, w, e, cfg.count, cfg.seed)
    g, code = upload_grid(grid, dev)
    r = torch.from_numpy(rows.astype(np.int32)).to(dev)
    c = torch.from_numpy(cols.astype(np.int32)).to(dev)
    return Signals(extract_rows(g, code, e, r, c, cfg.normalization, dtype))


def extract_patches(grid, cfg: PatchConfig) -> np.ndarray:
    """data.py:182-208 — a Fortran-ordered float64 (patch_edge^2, count) matrix."""
    sig = extract_patches_device(grid, cfg)
    return np.asfortranarray(sig.y.cpu().numpy().T)
