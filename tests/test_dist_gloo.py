"""Multi-rank host logic of the sharded iteration, world_size 2 over gloo (CPU).

The radix-select worst set, the threshold-tie split across ranks, the shard
ranges and the sharded initial sampling must reproduce the single-process
reference (sbo.py:223-228, 283-286) exactly.  The per-rank histogram here is the
numpy stand-in of the device kernel (sbo_key_histogram); on GPUs engine.py binds
the kernel and NCCL to the same functions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sbo_oracle as O
from paper_1412_4944_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, residual, w, cols, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = residual.shape[0]
        lo, hi = D.shard_range(m, world, rank)
        keys = D.key_of(residual[lo:hi])

        def allreduce(h):
            t = torch.from_numpy(np.ascontiguousarray(h))
            dist.all_reduce(t)
            return t.numpy()

        prefix, need_eq = D.select_threshold(lambda p, s: D.numpy_histogram(keys, p, s),
                                             allreduce, min(w, m))
        gt = keys > np.uint64(prefix)
        eq = keys == np.uint64(prefix)
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, torch.tensor([int(eq.sum())]))
        take = D.equal_quota([int(c.item()) for c in counts], rank, need_eq)
        eq_idx = np.nonzero(eq)[0][:take]
        members = np.sort(np.concatenate([np.nonzero(gt)[0], eq_idx])) + lo
        out[rank] = (members, D.local_members(cols, lo, hi) + lo)
    finally:
        dist.destroy_process_group()


def _run(residual, w, cols, world=2):
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, residual, w, cols, out), nprocs=world, join=True)
    return [out[r] for r in range(world)]


@pytest.mark.parametrize("w", [1, 37, 500, 999, 5000])
def test_distributed_worst_set_matches_reference(w):
    rng = np.random.default_rng(w)
    res = np.round(rng.random(3001), 2)  # heavy ties at the threshold
    res[::7] = 0.0
    cols = rng.choice(3001, size=256, replace=True)
    parts = _run(res, w, cols)
    got = np.sort(np.concatenate([p[0] for p in parts]))
    want = np.sort(O.worst_members(res, w))
    np.testing.assert_array_equal(got, want)
    # sharded sampling: the union of local members is the global sample (multiset)
    np.testing.assert_array_equal(np.sort(np.concatenate([p[1] for p in parts])), np.sort(cols))


def test_shard_ranges_cover_exactly():
    for m in (0, 1, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_single_rank_threshold_equals_sort():
    rng = np.random.default_rng(0)
    r = np.round(rng.random(5000), 3)
    keys = D.key_of(r)
    for w in (1, 10, 4999, 5000):
        prefix, need = D.select_threshold(lambda p, s: D.numpy_histogram(keys, p, s),
                                          lambda h: h, w)
        assert (keys > np.uint64(prefix)).sum() + need == w
        assert need <= (keys == np.uint64(prefix)).sum()
