"""The p = 256 sparse outer products (k_outer_sparse256 behind
sbo_outer_segments; onb.py:127-134 sparse_outer, P = Y X^T per block) against
numpy float64 on the same codes, for the representation's grouping (ragged
segments, signal order through a permutation) and a member list; and
determinism (the summation order is fixed: bit-identical reruns).

Contract: each P entry within 1e-14 of sum |y| |x| over its terms."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1412_4944_b200 import _lib as L  # noqa: E402
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402

P = 256


@pytest.fixture(scope="module")
def dev():
    return require_device()


def _blocks(K, seed):
    rng = np.random.default_rng(seed)
    return [np.linalg.qr(rng.standard_normal((P, P)))[0] for _ in range(K)]


def _outer(eng, g, n, order, idx, val):
    part = torch.full((g.max_seg, P, P), np.nan, dtype=torch.float64, device=eng.dev)
    L.call("sbo_outer_segments", eng.sig.y.data_ptr(), eng.sig.code, P,
           order.data_ptr() if order is not None else None, g.seg_lo.data_ptr(),
           g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg, eng.s0, max(n, 1),
           idx.data_ptr(), val.data_ptr(), part.data_ptr(), eng.stream)
    torch.cuda.synchronize()
    return part


def _check(part, g, rows, order, idx, val, k):
    lo, hi = g.seg_lo.cpu().numpy(), g.seg_hi.cpu().numpy()
    pt = part.cpu().numpy()
    ii, vv = idx.cpu().numpy().astype(np.int64), val.cpu().numpy()
    for s in range(int(g.nseg.item())):
        pos = np.arange(lo[s], hi[s])
        y = rows.astype(np.float64)[order[pos]]          # (n, 256)
        x = np.zeros((len(pos), P))
        xa = np.zeros((len(pos), P))
        for u in range(k):
            x[np.arange(len(pos)), ii[u, pos]] = vv[u, pos]
        xa = np.abs(x)
        want = y.T @ x
        bound = np.abs(y).T @ xa
        assert (np.abs(pt[s] - want) <= 1e-14 * bound + 1e-300).all(), s


@pytest.mark.parametrize("s0", [4, 16, 32])
def test_grouped_segments_match_numpy(dev, s0):
    rows = signals.patch_signals(5000 + 11, 16, 512, 512)
    eng = Engine(Signals.from_rows(rows, dev), s0, k_cap=3)
    eng.set_blocks(np.stack(_blocks(3, s0)))
    eng.represent_full()
    g = eng.group(eng.K)
    n, k = eng.m, eng.k
    idx = torch.zeros((k, n), dtype=torch.int16, device=dev)
    val = torch.zeros((k, n), dtype=torch.float64, device=dev)
    eng.code(g.perm, g, -1, False, n, idx, val)
    part = _outer(eng, g, n, g.perm, idx, val)
    _check(part, g, rows, g.perm.cpu().numpy().astype(np.int64), idx, val, k)
    again = _outer(eng, g, n, g.perm, idx, val)
    nseg = int(g.nseg.item())
    assert torch.equal(part[:nseg], again[:nseg])


def test_member_list_signed_values(dev):
    rng = np.random.default_rng(3)
    m = 2500
    rows = (rng.integers(0, 256, (m, P)) / 256.0 - 0.5).astype(np.float32)
    eng = Engine(Signals.from_rows(rows, dev), 16, k_cap=2)
    eng.set_blocks(np.stack(_blocks(2, 8)))
    members = torch.from_numpy(rng.permutation(m)[:1700].astype(np.int32)).to(dev)
    g = eng.list_segments(1700)
    idx = torch.zeros((16, 1700), dtype=torch.int16, device=dev)
    val = torch.zeros((16, 1700), dtype=torch.float64, device=dev)
    eng.code(members, g, 1, False, 1700, idx, val)
    part = _outer(eng, g, 1700, members, idx, val)
    _check(part, g, rows, members.cpu().numpy().astype(np.int64), idx, val, 16)
