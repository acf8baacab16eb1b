"""CPU oracle for the SBO iteration — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy/scipy restatement of the reference algorithm for the
hot path named in BASELINE.json (one Single-Block-Orthogonal dictionary-learning
iteration, arXiv 1412.4944).  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline / ``--impl reference``
leg may import it.  The product package ``paper_1412_4944_b200`` never imports
anything from here and has no CPU fallback.

Parity is pinned: ``tests/golden/make_golden.py`` runs the real reference
(``orthodict`` under /root/reference/pkg/src) on seeded inputs and commits the
outputs as fixtures; ``tests/test_oracle_golden.py`` checks this restatement
against them (decisions bit-exact, floats to 1e-12 relative).

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/orthodict/).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse

TILE = 256  # sbo.py:28-29 — fixed arithmetic tile of the representation pass
ORTHO_TOL = 1e-8  # onb.py:17
KINDS = ("squared-sum", "abs-sum")  # sbo.py:31


class OracleNumericalError(RuntimeError):
    """Orthonormality defect above ORTHO_TOL (onb.py:20-21, 119-124)."""


class OracleDecompositionError(RuntimeError):
    """SVD failed in both LAPACK drivers (linalg.py:15-16, 61-63)."""


# ----------------------------------------------------------------------------
# dense linear algebra  (linalg.py)
# ----------------------------------------------------------------------------

def canonical_signs(u: np.ndarray, vt: np.ndarray):
    """linalg.py:32-37 — flip (u_j, vt_j) so u_j's largest-|.| entry is >= 0."""
    r = u.shape[1]
    piv = np.abs(u).argmax(axis=0)
    neg = u[piv, np.arange(r)] < 0.0
    s = np.where(neg, -1.0, 1.0)
    return u * s, vt * s[:, None]


def svd(a: np.ndarray):
    """linalg.py:40-65 — thin SVD, gesdd with gesvd fallback, canonical signs.

    Returns (u, sigma, v) with v = vt.T (n x r)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or min(a.shape) < 1:
        raise ValueError(f"svd expects a nonempty 2-D matrix, got {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError("svd input contains NaN or Inf entries")
    try:
        u, s, vt = np.linalg.svd(a, full_matrices=False)
    except np.linalg.LinAlgError:
        try:
            u, s, vt = scipy.linalg.svd(a, full_matrices=False, lapack_driver="gesvd")
        except Exception as exc:  # pragma: no cover - LAPACK failure path
            raise OracleDecompositionError(
                f"SVD did not converge for a {a.shape[0]}x{a.shape[1]} matrix") from exc
    u, vt = canonical_signs(u, vt)
    return u, s, vt.T


def polar(pmat: np.ndarray) -> np.ndarray:
    """linalg.py:68-78 — orthogonal polar factor U V^T of a square P."""
    u, _, v = svd(pmat)
    return u @ v.T


def defect(q: np.ndarray) -> float:
    """linalg.py:81-86 — ||Q^T Q - I||_F."""
    g = q.T @ q
    return float(np.linalg.norm(g - np.eye(q.shape[1])))


def check_block(q: np.ndarray) -> None:
    """onb.py:119-124."""
    d = defect(q)
    if not np.isfinite(d) or d > ORTHO_TOL:
        raise OracleNumericalError(f"block lost orthonormality: defect {d:.3e} > 1e-08")


# ----------------------------------------------------------------------------
# single block (onb.py)
# ----------------------------------------------------------------------------

def top_support(coeffs: np.ndarray, s0: int):
    """onb.py:58-76 — keep the s0 largest |c| per column, ties -> lowest row.

    Returns (indices int64 (k, t) ascending per column, values (k, t))."""
    c = np.asarray(coeffs, dtype=np.float64)
    if c.ndim == 1:
        c = c[:, None]
    p = c.shape[0]
    k = min(s0, p)
    # a stable sort of -|c| keeps equal magnitudes in row order
    rows = np.argsort(-np.abs(c), axis=0, kind="stable")[:k]
    rows.sort(axis=0)
    return rows.astype(np.int64), np.take_along_axis(c, rows, axis=0)


def complete_basis(u: np.ndarray, rng) -> np.ndarray:
    """onb.py:98-116 — twice-projected Gram–Schmidt completion with seeded draws."""
    p, r = u.shape
    if r == p:
        return np.ascontiguousarray(u)
    rng = np.random.default_rng(0) if rng is None else rng
    basis = [u[:, j] for j in range(r)]
    while len(basis) < p:
        v = rng.standard_normal(p)
        for _ in range(2):
            for b in basis:
                v -= (b @ v) * b
        n = np.linalg.norm(v)
        if n >= 1e-8:
            basis.append(v / n)
    return np.column_stack(basis)


def init_block(ysub: np.ndarray, rng=None) -> np.ndarray:
    """onb.py:79-95 — U of the thin SVD, sigma > 1e-12*sigma_0 kept, completed."""
    ysub = np.asarray(ysub, dtype=np.float64)
    p = ysub.shape[0]
    if ysub.shape[1] == 0:
        return complete_basis(np.empty((p, 0)), rng)
    u, s, _ = svd(ysub)
    top = s[0] if s.size else 0.0
    keep = s > top * 1e-12 if top > 0.0 else np.zeros(s.shape, bool)
    q = complete_basis(u[:, keep], rng)
    check_block(q)
    return q


def outer_sparse(y: np.ndarray, idx: np.ndarray, val: np.ndarray) -> np.ndarray:
    """onb.py:127-134 — P = Y X^T with X given by per-column (rows, values)."""
    p, t = y.shape
    k = idx.shape[0]
    x = scipy.sparse.csc_array(
        (val.ravel(order="F"), idx.ravel(order="F"), np.arange(t + 1) * k), shape=(p, t))
    return np.asarray((x @ y.T).T)


def train_block(y: np.ndarray, q0: np.ndarray, s0: int, rounds: int, history=None):
    """onb.py:137-173 — R rounds of (select, P = Y X^T, Q = polar(P)).

    Returns (q, idx, val) with the final coding of the returned block.  When
    ``history`` is a list, each round's Q is appended (for round-by-round parity)."""
    y = np.asarray(y, dtype=np.float64)
    q = np.asarray(q0, dtype=np.float64)
    check_block(q)
    if y.shape[1] == 0:
        k = min(s0, q.shape[0])
        return q, np.empty((k, 0), np.int64), np.empty((k, 0))
    for _ in range(rounds):
        idx, val = top_support(q.T @ y, s0)
        q = polar(outer_sparse(y, idx, val))
        check_block(q)
        if history is not None:
            history.append(q.copy())
    idx, val = top_support(q.T @ y, s0)
    return q, idx, val


# ----------------------------------------------------------------------------
# union of blocks (sbo.py)
# ----------------------------------------------------------------------------

def energy_of(y: np.ndarray, q: np.ndarray, s0: int, kind: str = "squared-sum") -> float:
    """sbo.py:126-135 — one signal's hard-thresholded energy in one block."""
    c = np.abs(q.T @ np.asarray(y, dtype=np.float64).ravel())
    k = min(s0, c.size)
    top = np.sort(c)[c.size - k:]
    return float(top @ top) if kind == "squared-sum" else float(top.sum())


def _pool_map(fn, items, workers):
    items = list(items)
    if workers <= 1 or len(items) <= 1:
        return [fn(i) for i in items]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(fn, items))


@dataclass
class Coding:
    """Assignment + thresholded code of ``represent`` (sbo.py:61-78, onb.py:24-55)."""
    block: np.ndarray      # (m,) int64
    energy: np.ndarray     # (m,) f64, recomputed from the kept values
    residual_sq: np.ndarray  # (m,) f64
    indices: np.ndarray    # (k, m) int64
    values: np.ndarray     # (k, m) f64
    score: np.ndarray = field(default=None)  # (m,) f64 energy-pass score of the winner


def code_signals(y: np.ndarray, blocks, s0: int, kind: str = "squared-sum",
                 workers: int = 1) -> Coding:
    """sbo.py:138-220 — two-pass representation.

    Pass 1 (sbo.py:177-194), per fixed 256-column tile: C = tile^T [Q_0..Q_K-1],
    per (signal, block) the top-k of |C| scored by sum of squares or sum, argmax
    over blocks with the first maximum winning.  Pass 2 (sbo.py:196-218): the
    winners' codes by ``top_support`` grouped per block; energy and residual
    from the kept values."""
    y = np.asarray(y, dtype=np.float64)
    p, m = y.shape
    nb = len(blocks)
    k = min(s0, p)
    stacked = np.hstack(blocks)
    best = np.empty(m, np.int64)
    score = np.empty(m)
    norm2 = np.empty(m)

    def tile_pass(start):
        end = min(start + TILE, m)
        t = y[:, start:end]
        mags = np.abs(t.T @ stacked).reshape((end - start) * nb, p)
        mags.sort(axis=1)
        top = mags[:, p - k:]
        e = np.einsum("ij,ij->i", top, top) if kind == "squared-sum" else top.sum(axis=1)
        e = e.reshape(end - start, nb)
        best[start:end] = e.argmax(axis=1)
        score[start:end] = e.max(axis=1)
        norm2[start:end] = np.einsum("ij,ij->j", t, t)

    _pool_map(tile_pass, range(0, m, TILE), workers)

    indices = np.empty((k, m), np.int64)
    values = np.empty((k, m))
    order = np.argsort(best, kind="stable")
    cuts = np.searchsorted(best[order], np.arange(nb + 1))

    def winner_pass(b):
        cols = order[cuts[b]:cuts[b + 1]]
        if cols.size:
            i, v = top_support(blocks[b].T @ y[:, cols], s0)
            indices[:, cols] = i
            values[:, cols] = v

    _pool_map(winner_pass, range(nb), workers)
    kept2 = np.einsum("ij,ij->j", values, values)
    energy = kept2 if kind == "squared-sum" else np.abs(values).sum(axis=0)
    resid = np.maximum(norm2 - kept2, 0.0)
    return Coding(best, energy, resid, indices, values, score)


def worst_members(residual_sq: np.ndarray, w: int) -> np.ndarray:
    """sbo.py:223-228 — the w largest residuals, descending, ties -> low index."""
    if w < 1:
        raise ValueError(f"worst-set size must be at least 1, got {w}")
    order = np.argsort(-np.asarray(residual_sq), kind="stable")
    return order[:min(w, order.size)]


def group_order(block: np.ndarray, nb: int):
    """sbo.py:231-249 — stable permutation by block and per-block [start, end)."""
    perm = np.argsort(block, kind="stable")
    cuts = np.searchsorted(block[perm], np.arange(nb + 1))
    return perm, [(int(cuts[b]), int(cuts[b + 1])) for b in range(nb)]


def stream(seed: int, phase: int, ordinal: int) -> np.random.Generator:
    """sbo.py:252-256 — independent seeded stream per (phase, block ordinal)."""
    ss = np.random.SeedSequence([int(seed) & 0xFFFFFFFFFFFFFFFF, phase, ordinal])
    return np.random.default_rng(ss)


def initial_blocks(y, s0, k0, p0, rounds, seed, workers=1):
    """sbo.py:259-292 — k0 blocks, each init_block + train_block on p0 samples."""
    y = np.asarray(y, dtype=np.float64)
    m = y.shape[1]
    replace = p0 > m

    def one(b):
        rng = stream(seed, 0, b)
        cols = rng.choice(m, size=p0, replace=replace)
        ysub = y[:, cols]
        q, _, _ = train_block(ysub, init_block(ysub, rng), s0, rounds)
        return q

    return _pool_map(one, range(k0), workers)


def rmse_of(residual_sq: np.ndarray, p: int, m: int) -> float:
    """sbo.py:295-296."""
    return math.sqrt(max(float(residual_sq.sum()), 0.0) / (p * m))


@dataclass
class IterationTrace:
    """Everything one teacher-forced SBO iteration produces (sbo.py:352-397)."""
    worst: np.ndarray
    new_block: np.ndarray
    rep1: Coding
    perm: np.ndarray
    ranges: list
    blocks: list  # after retraining
    empty: list   # block ids left unchanged
    rep2: Coding
    rmse: float


def iterate(y, blocks, residual_sq, s0, rounds, w, seed, kind="squared-sum", workers=1,
            rng=None) -> IterationTrace:
    """sbo.py:352-397 — ONE SBO iteration from an entering (blocks, residuals).

    ``blocks`` is not modified; a new list is returned in the trace."""
    y = np.asarray(y, dtype=np.float64)
    p, m = y.shape
    blocks = [b.copy() for b in blocks]
    worst = worst_members(residual_sq, w)
    rng = stream(seed, 1, len(blocks)) if rng is None else rng
    ysub = y[:, worst]
    q_new, _, _ = train_block(ysub, init_block(ysub, rng), s0, rounds)
    blocks.append(q_new)
    rep1 = code_signals(y, blocks, s0, kind, workers)
    perm, ranges = group_order(rep1.block, len(blocks))
    grouped = y[:, perm]

    def retrain(b):
        lo, hi = ranges[b]
        if lo == hi:
            return None
        return train_block(grouped[:, lo:hi], blocks[b], s0, rounds)[0]

    empty = []
    for b, q in enumerate(_pool_map(retrain, range(len(blocks)), workers)):
        if q is None:
            empty.append(b)
        else:
            blocks[b] = q
    rep2 = code_signals(y, blocks, s0, kind, workers)
    return IterationTrace(worst, q_new, rep1, perm, ranges, blocks, empty, rep2,
                          rmse_of(rep2.residual_sq, p, m))


def train(y, s0, k0=5, p0=4096, rounds=6, worst_size=None, k_max=64, target_error=0.0,
          kind="squared-sum", seed=0, workers=1):
    """sbo.py:299-420 — the full training loop; returns (blocks, coding, rmses, notes)."""
    y = np.asarray(y, dtype=np.float64)
    p, m = y.shape
    w = worst_size if worst_size is not None else max(p, m // 16)
    blocks = initial_blocks(y, s0, k0, p0, rounds, seed, workers)
    rep = code_signals(y, blocks, s0, kind, workers)
    rmse = rmse_of(rep.residual_sq, p, m)
    rmses, notes = [rmse], []
    while rmse > target_error and len(blocks) < k_max:
        it = len(rmses)
        tr = iterate(y, blocks, rep.residual_sq, s0, rounds, w, seed, kind, workers)
        notes += [f"iteration {it}: block {b} had no signals, left unchanged" for b in tr.empty]
        blocks, rep, rmse = tr.blocks, tr.rep2, tr.rmse
        rmses.append(rmse)
    return blocks, rep, rmses, notes


def frob_error(y, blocks, block, indices, values) -> float:
    """linalg.py:89-102, 148-162 — ||Y - D X||_F for a single-best-block code."""
    y = np.asarray(y, dtype=np.float64)
    yhat = np.zeros_like(y)
    for b, q in enumerate(blocks):
        cols = np.nonzero(block == b)[0]
        for r in range(indices.shape[0]):
            yhat[:, cols] += q[:, indices[r, cols]] * values[r, cols]
    return float(np.linalg.norm(y - yhat))


def default_workers() -> int:
    """parallel.py:16-29 (ORTHODICT_WORKERS or the CPU count)."""
    env = os.environ.get("ORTHODICT_WORKERS")
    return int(env) if env else (os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# signal ingestion
# ---------------------------------------------------------------------------

def pairwise_sum_rows(a: np.ndarray) -> np.ndarray:
    """Column sums of a (n, count) float64 array in numpy's pairwise order
    (numpy umath loops_utils.h.src, pairwise_sum; the reduction data.py:207's
    ``mean(axis=0)`` runs over each contiguous column): plain accumulation below
    8 terms, 8 interleaved accumulators up to 128, halving (multiples of 8) above."""
    n = a.shape[0]
    if n < 8:
        res = np.zeros(a.shape[1:], np.float64)
        for i in range(n):
            res = res + a[i]
        return res
    if n <= 128:
        r = [a[j].copy() for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = r[j] + a[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res = res + a[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum_rows(a[:n2]) + pairwise_sum_rows(a[n2:])


def extract_patches(grid: np.ndarray, edge: int, count: int, seed: int,
                    normalization: str = "unit-range") -> np.ndarray:
    """data.py:182-208 — Fortran (edge^2, count) float64 signals of random patches:
    corners from default_rng(seed).integers (rows, then columns; data.py:199-201),
    column-major vectorization (entry (r, c) at c*edge + r; data.py:203-204), /255
    (data.py:205), minus the patch mean for the dc-removed variant (data.py:206-207)."""
    grid = np.asarray(grid)
    h, w = grid.shape
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, h - edge + 1, size=count)
    cols = rng.integers(0, w - edge + 1, size=count)
    n = edge * edge
    y = np.empty((n, count), np.float64)
    for c in range(edge):
        for r in range(edge):
            y[c * edge + r] = grid[rows + r, cols + c].astype(np.float64) / 255.0
    if normalization == "unit-range-dc-removed":
        y = y - pairwise_sum_rows(y) / n
    return np.asfortranarray(y)
