"""Single orthonormal block (1ONB, Alg. 1) on the device (mirror of orthodict.onb).

Same names, argument meaning and exceptions as onb.py:17-173; the coding step,
the sparse outer product and the polar update run in the sm_100a library.
"""
from __future__ import annotations

import copy
from dataclasses import dataclass

import numpy as np
import scipy.sparse
import torch

from . import _lib as L

ORTHONORMALITY_TOL = 1e-8  # onb.py:17


class NumericalError(RuntimeError):
    """A trained block violated its orthonormality contract (onb.py:20-21)."""


@dataclass
class ThresholdedCode:
    """Per-column kept rows (strictly increasing) and values (onb.py:24-55)."""

    indices: np.ndarray  # (k, m) int64
    values: np.ndarray   # (k, m) float64

    @property
    def nnz_per_column(self) -> int:
        return self.indices.shape[0]

    @property
    def num_columns(self) -> int:
        return self.indices.shape[1]

    def to_csc(self, p: int) -> scipy.sparse.csc_array:
        k, m = self.indices.shape
        return scipy.sparse.csc_array(
            (self.values.ravel(order="F"), self.indices.ravel(order="F"),
             np.arange(m + 1, dtype=np.int64) * k), shape=(p, m))


def _dev():
    from .engine import require_device
    return require_device()


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def select_top(coeffs: np.ndarray, s0: int) -> ThresholdedCode:
    """onb.py:58-76 — the s0 largest |c| per column, ties toward the lowest row."""
    if s0 < 1:
        raise ValueError(f"s0 must be at least 1, got {s0}")
    c = np.asarray(coeffs, dtype=np.float64)
    if c.ndim == 1:
        c = c[:, None]
    p, t = c.shape
    k = min(s0, p)
    if p > 256:
        raise ValueError("select_top on the device supports up to 256 rows")
    dev = _dev()
    rows = torch.from_numpy(np.ascontiguousarray(c.T)).to(dev)
    idx = torch.empty((k, max(t, 1)), dtype=torch.int16, device=dev)
    val = torch.empty((k, max(t, 1)), dtype=torch.float64, device=dev)
    L.call("sbo_select_top", rows.data_ptr(), t, p, s0, max(t, 1), idx.data_ptr(),
           val.data_ptr(), _stream(dev))
    return ThresholdedCode(idx[:, :t].cpu().numpy().astype(np.int64), val[:, :t].cpu().numpy())


def _check_block(q: np.ndarray) -> None:
    """onb.py:119-124."""
    from .linalg import orthonormality_defect
    d = orthonormality_defect(q)
    if not np.isfinite(d) or d > ORTHONORMALITY_TOL:
        raise NumericalError(
            f"block lost orthonormality: defect {d:.3e} > {ORTHONORMALITY_TOL:.0e}")


def init_onb(ysub: np.ndarray, rng: np.random.Generator | None = None) -> np.ndarray:
    """onb.py:79-116 — U of the thin SVD of ysub (sigma > 1e-12 sigma_0 kept), completed
    by twice-projected Gram–Schmidt on draws from ``rng`` (default_rng(0) when None).

    The device computes the float64 Gram matrix and its Jacobi eigenvectors; the
    caller's generator advances by exactly the draws the completion consumed."""
    from .engine import Engine, Signals
    from .linalg import DecompositionError

    ysub = np.asarray(ysub, dtype=np.float64)
    if ysub.ndim != 2:
        raise ValueError(f"expected a 2-D sample, got shape {ysub.shape}")
    if not np.isfinite(ysub).all():
        raise ValueError("thin_svd input contains NaN or Inf entries")
    p, t = ysub.shape
    rng = np.random.default_rng(0) if rng is None else rng
    draws = copy.deepcopy(rng).standard_normal((p + 8, p))
    dev = _dev()
    if t:
        eng = Engine(Signals.from_reference(ysub, dev), 1, k_cap=1)
        G = eng.gram(None, t)
    else:
        eng = Engine(Signals(torch.zeros((1, p), dtype=torch.float64, device=dev)), 1, k_cap=1)
        G = torch.zeros((p, p), dtype=torch.float64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    rank = torch.zeros(2, dtype=torch.int32, device=dev)
    eng.init_block(G, t, draws, 0, st, rank)
    status, used = int(st.item()) & 0xFF, int(rank[1].item())
    if status == L.ST_NOCONV:
        raise DecompositionError(f"SVD did not converge for a {p}x{t} matrix")
    if used:
        rng.standard_normal((used, p))  # advance the caller's stream like the reference
    q = eng.blocks[0].cpu().numpy()
    if status == L.ST_DEFECT:
        _check_block(q)
    return q


def sparse_outer(y: np.ndarray, code: ThresholdedCode) -> np.ndarray:
    """onb.py:127-134 — P = Y X^T with X in thresholded form, never densified."""
    from .engine import Engine, Signals

    y = np.asarray(y, dtype=np.float64)
    idx, val = np.asarray(code.indices), np.asarray(code.values, dtype=np.float64)
    if idx.shape[1] != y.shape[1]:
        raise ValueError(f"code covers {idx.shape[1]} signals but the matrix has {y.shape[1]}")
    p, t = y.shape
    dev = _dev()
    if t == 0:
        return np.zeros((p, p))
    eng = Engine(Signals.from_reference(y, dev), idx.shape[0], k_cap=1)
    g = eng.list_segments(t)
    I = torch.from_numpy(np.ascontiguousarray(idx.astype(np.int16))).to(dev)
    V = torch.from_numpy(np.ascontiguousarray(val)).to(dev)
    partial = torch.empty((g.max_seg, p, p), dtype=torch.float64, device=dev)
    P = torch.empty((1, p, p), dtype=torch.float64, device=dev)
    L.call("sbo_outer_segments", eng.sig.y.data_ptr(), eng.sig.code, p, None,
           g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg,
           idx.shape[0], t, I.data_ptr(), V.data_ptr(), partial.data_ptr(), _stream(dev))
    L.call("sbo_reduce_segments", partial.data_ptr(), None, g.nseg.data_ptr(), g.max_seg, 1,
           p, P.data_ptr(), _stream(dev))
    return P[0].cpu().numpy()


def train_onb(y: np.ndarray, q0: np.ndarray, s0: int, rounds: int
              ) -> tuple[np.ndarray, ThresholdedCode]:
    """onb.py:137-173 — ``rounds`` passes of (select_top(Q^T Y), P = Y X^T, Q = polar(P)),
    then the coding of the final block."""
    from .engine import Engine, Signals, check_status

    y = np.asarray(y, dtype=np.float64)
    q = np.asarray(q0, dtype=np.float64)
    if q.ndim != 2 or q.shape[0] != q.shape[1]:
        raise ValueError(f"initial block must be square, got {q.shape}")
    if y.shape[0] != q.shape[0]:
        raise ValueError(
            f"signals have dimension {y.shape[0]} but the block is {q.shape[0]}x{q.shape[1]}")
    if rounds < 0:
        raise ValueError(f"rounds must be nonnegative, got {rounds}")
    if not np.isfinite(y).all():
        raise ValueError("signal matrix contains NaN or Inf entries")
    if s0 < 1:
        raise ValueError(f"s0 must be at least 1, got {s0}")
    _check_block(q)
    p, t = y.shape
    k = min(s0, p)
    if t == 0:
        return q, ThresholdedCode(np.empty((k, 0), np.int64), np.empty((k, 0)))
    dev = _dev()
    eng = Engine(Signals.from_reference(y, dev), s0, k_cap=1)
    eng.set_blocks(q[None])
    g = eng.list_segments(t)
    st = torch.zeros((max(rounds, 1), 1), dtype=torch.int32, device=dev)
    eng.train_rounds(None, g, t, rounds, 1, 0, None, st, single=True)
    idx = torch.empty((k, t), dtype=torch.int16, device=dev)
    val = torch.empty((k, t), dtype=torch.float64, device=dev)
    eng.code(None, g, 0, True, t, idx, val)
    check_status(st.cpu().numpy()[:rounds], p)
    return (eng.blocks[0].cpu().numpy(),
            ThresholdedCode(idx.cpu().numpy().astype(np.int64), val.cpu().numpy()))
