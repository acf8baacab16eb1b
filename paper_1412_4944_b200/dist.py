"""Host logic of the signal-sharded (multi-GPU) SBO iteration.

Signals are split into contiguous column shards, one per rank (rank r owns
global signals [r*m/n, (r+1)*m/n) — SURVEY.md §8e).  Everything per-signal stays
local; the exchanges are:

  * worst set (sbo.py:223-228): a radix select over the float64 residual keys
    with a 256-bin histogram allreduce per 8-bit digit, then threshold ties
    taken in global signal order (lower ranks first) — ``select_threshold`` and
    ``equal_quota``;
  * the p x p Gram matrix of the worst set and, per 1ONB round, the p x p
    matrices P_b = Y_b X_b^T of every block: float64 allreduce (sum);
  * initial sampling (sbo.py:283-286): every rank draws the same global columns
    and keeps its own (``local_members``);
  * the residual sum for the RMSE: a scalar allreduce.

The functions here are pure host code over callables, so the same logic runs
on GPUs (engine.py binds the device histogram/collect kernels and NCCL) and in
the CPU multi-process tests (gloo with numpy stand-ins).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def key_of(residual: np.ndarray) -> np.ndarray:
    """Order-preserving uint64 keys of nonnegative float64 residuals (as on the device)."""
    r = np.asarray(residual, dtype=np.float64)
    k = r.view(np.uint64).copy()
    k[~(r > 0.0)] = 0
    return k


def select_threshold(hist: Callable[[int, int], np.ndarray],
                     allreduce: Callable[[np.ndarray], np.ndarray], need: int):
    """MSB-first radix select of the need-th largest key over all ranks.

    ``hist(prefix, shift)`` returns this rank's 256-bin histogram of digit
    ``(key >> shift) & 255`` among keys whose bits above shift+8 equal prefix's.
    Returns (threshold_key, need_equal): the members are every key above the
    threshold plus ``need_equal`` keys equal to it (lowest global index first)."""
    prefix = 0
    for shift in range(56, -8, -8):
        h = np.asarray(allreduce(np.asarray(hist(prefix, shift), dtype=np.int64)))
        cum, digit = 0, 0
        for d in range(255, -1, -1):
            if cum + int(h[d]) >= need:
                digit = d
                break
            cum += int(h[d])
        need -= cum
        prefix |= digit << shift
    return prefix, need


def equal_quota(equal_counts: list[int], rank: int, need_equal: int) -> int:
    """Threshold-equal members this rank keeps: ties go to the lowest global
    indices, i.e. to lower ranks first under contiguous column sharding."""
    before = sum(equal_counts[:rank])
    return max(0, min(equal_counts[rank], need_equal - before))


def shard_range(m_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous column shard of rank (sizes differ by at most one)."""
    base, extra = divmod(m_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def local_members(cols: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """This shard's part of a global column sample, as local indices, in sample order."""
    cols = np.asarray(cols)
    sel = cols[(cols >= lo) & (cols < hi)]
    return (sel - lo).astype(np.int64)


def numpy_histogram(keys: np.ndarray, prefix: int, shift: int) -> np.ndarray:
    """Reference implementation of the device key histogram (tests / CPU ranks)."""
    keys = np.asarray(keys, dtype=np.uint64)
    if shift + 8 < 64:
        keys = keys[(keys >> np.uint64(shift + 8)) == (np.uint64(prefix) >> np.uint64(shift + 8))]
    digits = ((keys >> np.uint64(shift)) & np.uint64(255)).astype(np.int64)
    return np.bincount(digits, minlength=256).astype(np.int64)
