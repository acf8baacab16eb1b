"""Dense linear algebra of the SBO path on the device (mirror of orthodict.linalg).

Same names, argument meaning and exceptions as the reference module
(linalg.py:15-162); the arithmetic runs in the sm_100a library:
``thin_svd`` -> sbo_svd (one-sided Jacobi, float64), ``procrustes_polar`` ->
sbo_polar, ``orthonormality_defect`` -> sbo_defect, ``frobenius_error`` ->
sbo_frobenius_sq (union-of-blocks codes).
"""
from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _lib as L


class DecompositionError(RuntimeError):
    """A matrix decomposition failed to converge (linalg.py:15-16)."""


class SvdResult(NamedTuple):
    """Thin SVD ``A = u @ diag(sigma) @ v.T`` with canonical column signs (linalg.py:19-29)."""

    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray


def _dev():
    from .engine import require_device
    return require_device()


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def thin_svd(a: np.ndarray) -> SvdResult:
    """linalg.py:40-65 — thin SVD, sigma descending, each u column's largest entry >= 0."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"thin_svd expects a nonempty 2-D matrix, got shape {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError("thin_svd input contains NaN or Inf entries")
    p, n = a.shape
    wide = n > p
    m = a.T if wide else a          # rows >= cols
    rows, cols = m.shape
    dev = _dev()
    M = torch.from_numpy(np.ascontiguousarray(m)).to(dev)
    U = torch.empty((rows, cols), dtype=torch.float64, device=dev)
    S = torch.empty(cols, dtype=torch.float64, device=dev)
    V = torch.empty((cols, cols), dtype=torch.float64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(L.size("sbo_svd_workspace_bytes", rows, cols), dtype=torch.uint8, device=dev)
    L.call("sbo_svd", M.data_ptr(), rows, cols, U.data_ptr(), S.data_ptr(), V.data_ptr(),
           st.data_ptr(), ws.data_ptr(), ws.numel(), _stream(dev))
    if int(st.item()) != L.ST_OK:
        raise DecompositionError(f"SVD did not converge for a {p}x{n} matrix")
    u, s, v = U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy()
    if not wide:
        return SvdResult(u, s, v)
    # a^T = u s v^T  ->  a = v s u^T; re-apply the sign convention on the new u
    uu, vv = v, u
    piv = np.abs(uu).argmax(axis=0)
    sg = np.where(uu[piv, np.arange(uu.shape[1])] < 0.0, -1.0, 1.0)
    return SvdResult(uu * sg, s, vv * sg)


def procrustes_polar(p_mat: np.ndarray) -> np.ndarray:
    """linalg.py:68-78 — orthogonal Q maximizing trace(Q^T P), Q = U V^T."""
    p_mat = np.asarray(p_mat, dtype=np.float64)
    if p_mat.ndim != 2 or p_mat.shape[0] != p_mat.shape[1]:
        raise ValueError(f"procrustes_polar expects a square matrix, got {p_mat.shape}")
    if not np.isfinite(p_mat).all():
        raise ValueError("thin_svd input contains NaN or Inf entries")
    p = p_mat.shape[0]
    dev = _dev()
    P = torch.from_numpy(np.ascontiguousarray(p_mat)).to(dev)
    Q = torch.empty((p, p), dtype=torch.float64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(L.size("sbo_polar_workspace_bytes", 1, p), dtype=torch.uint8, device=dev)
    L.call("sbo_polar", P.data_ptr(), 1, p, None, Q.data_ptr(), None, None, st.data_ptr(),
           ws.data_ptr(), ws.numel(), _stream(dev))
    if int(st.item()) & 0xFF == L.ST_NOCONV:
        raise DecompositionError(f"SVD did not converge for a {p}x{p} matrix")
    return Q.cpu().numpy()


def orthonormality_defect(q: np.ndarray) -> float:
    """linalg.py:81-86 — ||Q^T Q - I||_F (square blocks)."""
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 2 or q.shape[0] != q.shape[1]:
        raise ValueError(f"orthonormality_defect expects a square block, got {q.shape}")
    dev = _dev()
    Q = torch.from_numpy(np.ascontiguousarray(q)).to(dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    L.call("sbo_defect", Q.data_ptr(), 1, q.shape[0], out.data_ptr(), _stream(dev))
    return float(out.item())


def frobenius_error(y: np.ndarray, dictionary, code) -> float:
    """linalg.py:89-102 — ||Y - D X||_F for a union dictionary with a single-best-block
    code, or a single orthonormal block with a thresholded code (the SBO path's pairings)."""
    from .engine import Signals
    from .sbo import SparseCode, UnionDictionary

    y = np.asarray(y, dtype=np.float64)
    if y.ndim != 2:
        raise ValueError(f"expected a 2-D signal matrix, got shape {y.shape}")
    p, m = y.shape
    if isinstance(dictionary, UnionDictionary):
        if not isinstance(code, SparseCode):
            raise ValueError("a union dictionary needs a single-best-block code")
        blocks = np.stack(dictionary.blocks)
        block = np.asarray(code.block)
    else:
        d = np.asarray(dictionary, dtype=np.float64)
        if d.ndim != 2 or d.shape != (p, p) or not hasattr(code, "indices"):
            raise NotImplementedError(
                "frobenius_error on the device covers the SBO pairings (union of blocks with a "
                "single-best-block code, or one p x p block with a thresholded code)")
        blocks = d[None]
        block = np.zeros(np.asarray(code.indices).shape[1], np.int64)
    idx, val = np.asarray(code.indices), np.asarray(code.values, dtype=np.float64)
    if idx.shape != val.shape or idx.shape[1] != m:
        raise ValueError(f"reconstruction shape ({p}, {idx.shape[1]}) != signals {y.shape}")
    # range checks on the host (the device kernel indexes blocks[block[j]] and
    # q[:, idx] directly): like the reference's block loop (linalg.py:148-158),
    # a signal whose block id is outside [0, K) is never reconstructed (its
    # approximation is zero); atom indices follow numpy indexing — negative ones
    # wrap, out-of-range ones raise IndexError
    block = np.asarray(block, dtype=np.int64)
    live = (block >= 0) & (block < blocks.shape[0])
    if not live.all():
        val = np.where(live[None, :], val, 0.0)
        block = np.where(live, block, 0)
    idx = np.asarray(idx, dtype=np.int64)
    used = idx[:, live]
    if used.size and (used.min() < -p or used.max() >= p):
        bad = int(used.max()) if used.max() >= p else int(used.min())
        raise IndexError(f"index {bad} is out of bounds for axis 1 with size {p}")
    idx = np.where(live[None, :], idx % p, 0)
    dev = _dev()
    sig = Signals.from_reference(y, dev)
    B = torch.from_numpy(np.ascontiguousarray(blocks)).to(dev)
    blk = torch.from_numpy(block.astype(np.int32)).to(dev)
    I = torch.from_numpy(np.ascontiguousarray(idx.astype(np.int16))).to(dev)
    Vv = torch.from_numpy(np.ascontiguousarray(val)).to(dev)
    tot = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = torch.empty(8 * (m // 8 + 2), dtype=torch.uint8, device=dev)
    L.call("sbo_frobenius_sq", sig.y.data_ptr(), sig.code, m, p, B.data_ptr(), blk.data_ptr(),
           idx.shape[0], m, I.data_ptr(), Vv.data_ptr(), tot.data_ptr(), ws.data_ptr(),
           ws.numel(), _stream(dev))
    return float(np.sqrt(max(tot.item(), 0.0)))
