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


def _p_i8_256(eng, g, n, order, nblocks, idx, val, seg_block):
    """P per block from the tensor-core product on the 16 (64-dim, 64-atom) slices
    (sbo_outer_i8_segments, p = 256) and from the sparse float64 kernel +
    ordered reduction, on the same codes."""
    st, ld = eng.stream, max(n, 1)
    order_p = order.data_ptr() if order is not None else None
    tiles = torch.empty(L.size("sbo_y_tiles_bytes", n, g.max_seg, P), dtype=torch.uint8,
                        device=eng.dev)
    L.call("sbo_y_tiles", eng.ydig.data_ptr(), P, order_p, g.seg_lo.data_ptr(),
           g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg, tiles.data_ptr(), st)
    ws = torch.empty(L.size("sbo_outer_i8_workspace_bytes", nblocks, P), dtype=torch.uint8,
                     device=eng.dev)
    p_i8 = torch.zeros((nblocks, P, P), dtype=torch.float64, device=eng.dev)
    L.call("sbo_outer_i8_segments", tiles.data_ptr(), P,
           seg_block.data_ptr() if seg_block is not None else None, g.seg_lo.data_ptr(),
           g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg, nblocks, eng.s0, ld,
           idx.data_ptr(), val.data_ptr(), eng.i8[0], eng.i8[1], p_i8.data_ptr(),
           ws.data_ptr(), ws.numel(), st)
    part = _outer(eng, g, n, order, idx, val)
    p_f64 = torch.zeros_like(p_i8)
    L.call("sbo_reduce_segments", part.data_ptr(),
           seg_block.data_ptr() if seg_block is not None else None, g.nseg.data_ptr(),
           g.max_seg, nblocks, P, p_f64.data_ptr(), st)
    torch.cuda.synchronize()
    return p_i8.cpu().numpy(), p_f64.cpu().numpy()


def _close(pi, pf):
    for b in range(pf.shape[0]):
        scale = max(np.abs(pf[b]).max(), 1e-300)
        assert np.abs(pi[b] - pf[b]).max() <= 1e-13 * scale, (b, np.abs(pi[b] - pf[b]).max())


@pytest.mark.parametrize("s0", [4, 16, 32])
def test_i8_256_products_grouped(dev, s0, monkeypatch):
    monkeypatch.setenv("SBO_I8", "1")
    monkeypatch.setenv("SBO_CI8", "1")
    rows = signals.patch_signals(6000 + 11, 16, 512, 512)
    eng = Engine(Signals.from_rows(rows, dev), s0, k_cap=4)
    eng.set_blocks(np.stack(_blocks(4, s0 + 1)))
    assert eng.i8 is not None and eng.ci8
    eng.represent_full()
    g = eng.group(eng.K)
    n, k = eng.m, eng.k
    idx = torch.zeros((k, n), dtype=torch.int16, device=dev)
    val = torch.zeros((k, n), dtype=torch.float64, device=dev)
    eng.code(g.perm, g, -1, False, n, idx, val)
    pi, pf = _p_i8_256(eng, g, n, g.perm, eng.K, idx, val, g.seg_block)
    _close(pi, pf)


def test_i8_256_products_member_list_signed(dev, monkeypatch):
    monkeypatch.setenv("SBO_I8", "1")
    monkeypatch.setenv("SBO_CI8", "1")
    rng = np.random.default_rng(5)
    m = 2500
    rows = (rng.integers(0, 256, (m, P)) / 256.0 - 0.5).astype(np.float32)
    rows[rng.random(m) < 0.1] = 0.0
    eng = Engine(Signals.from_rows(rows, dev), 16, k_cap=2)
    eng.set_blocks(np.stack(_blocks(2, 9)))
    assert eng.i8 is not None
    members = torch.from_numpy(rng.permutation(m)[:1700].astype(np.int32)).to(dev)
    g = eng.list_segments(1700)
    idx = torch.zeros((16, 1700), dtype=torch.int16, device=dev)
    val = torch.zeros((16, 1700), dtype=torch.float64, device=dev)
    eng.code(members, g, 1, False, 1700, idx, val)
    pi, pf = _p_i8_256(eng, g, 1700, members, 1, idx, val, None)
    _close(pi, pf)
