"""The round's coding / residual pass on tcgen05 from exact integer digits
(round_i8.cu; onb.py:170-171 select_top(Q^T Y), sbo.py:207-218) against the
float64 DMMA kernels and the CPU oracle on the same signals and blocks.

Contract: supports bit-exact (ties -> lower atom, oracle.top_support), values
to 1e-14 of ||y|| (the digit projection and the float64 projection each sit
within ~1e-16 ||y|| of the exact product), residuals / scores to 1e-13 of
||y||^2."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import sbo_oracle as O  # noqa: E402
from paper_1412_4944_b200 import _lib as L  # noqa: E402
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    return require_device()


@pytest.fixture(autouse=True)
def _i8_on(monkeypatch):
    monkeypatch.setenv("SBO_I8", "1")
    monkeypatch.setenv("SBO_RI8", "1")


def _engine(dev, rows, blocks, s0):
    eng = Engine(Signals.from_rows(rows, dev), s0, k_cap=len(blocks))
    eng.set_blocks(np.stack(blocks))
    assert eng.i8 is not None and eng.ri8
    return eng


def _random_blocks(K, seed):
    rng = np.random.default_rng(seed)
    return [np.linalg.qr(rng.standard_normal((64, 64)))[0] for _ in range(K)]


def _ri8(eng, g, n, order, mode, override=-1, nblocks=None):
    k, ld, st = eng.k, max(n, 1), eng.stream
    nb = nblocks or eng.K
    ws = torch.empty(L.size("sbo_round_i8_workspace_bytes", nb), dtype=torch.uint8,
                     device=eng.dev)
    idx = torch.full((k, ld), -7, dtype=torch.int16, device=eng.dev)
    val = torch.full((k, ld), np.nan, dtype=torch.float64, device=eng.dev)
    rest = torch.full((eng.m,), np.nan, dtype=torch.float64, device=eng.dev)
    score = torch.full((eng.m,), np.nan, dtype=torch.float64, device=eng.dev)
    L.call("sbo_round_i8_segments", eng.ydig.data_ptr(), eng.i8[0],
           order.data_ptr() if order is not None else None, g.seg_block.data_ptr(),
           g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg,
           eng.blocks.data_ptr(), nb, override, eng.s0, mode, eng.kind, ld,
           idx.data_ptr() if mode == 0 else None, val.data_ptr() if mode == 0 else None,
           rest.data_ptr() if mode == 1 else None, score.data_ptr() if mode == 1 else None,
           ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize()
    return idx, val, rest, score


def _dmma_codes(eng, g, n, order, override=-1):
    k, ld = eng.k, max(n, 1)
    idx = torch.zeros((k, ld), dtype=torch.int16, device=eng.dev)
    val = torch.zeros((k, ld), dtype=torch.float64, device=eng.dev)
    L.call("sbo_round_code_segments", eng.sig.y.data_ptr(), eng.sig.code, 64,
           order.data_ptr() if order is not None else None, g.seg_block.data_ptr(),
           g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg,
           eng.blocks.data_ptr(), override, eng.s0, ld, idx.data_ptr(), val.data_ptr(),
           eng.stream)
    torch.cuda.synchronize()
    return idx, val


def _oracle_codes(rows, blocks, block_of_pos, order, s0):
    """top_support of the float64 projection of each position's signal in its block."""
    y = rows.astype(np.float64)[order]                     # (n, 64), segment order
    idx = np.empty((min(s0, 64), len(order)), np.int64)
    val = np.empty(idx.shape)
    for b in np.unique(block_of_pos):
        sel = np.nonzero(block_of_pos == b)[0]
        c = blocks[b].T @ y[sel].T                           # (64, n_b)
        i, v = O.top_support(c, s0)
        idx[:, sel], val[:, sel] = i, v
    return idx, val


def _block_of_positions(g, n):
    lo, hi = g.seg_lo.cpu().numpy(), g.seg_hi.cpu().numpy()
    sb = g.seg_block.cpu().numpy()
    out = np.empty(n, np.int64)
    for s in range(int(g.nseg.item())):
        out[lo[s]:hi[s]] = sb[s]
    return out


@pytest.mark.parametrize("s0", [4, 8, 16, 32])
def test_codes_match_oracle_and_dmma(dev, s0):
    """Unit-range patches, 5 random blocks, the representation's grouping
    (ragged per-block tails)."""
    rows = signals.patch_signals(20000 + 37, 8, 512, 512)
    blocks = _random_blocks(5, s0)
    eng = _engine(dev, rows, blocks, s0)
    eng.represent_full()
    g = eng.group(eng.K)
    idx, val, _, _ = _ri8(eng, g, eng.m, g.perm, 0)
    order = g.perm.cpu().numpy().astype(np.int64)
    oi, ov = _oracle_codes(rows, blocks, _block_of_positions(g, eng.m), order, s0)
    gi = idx.cpu().numpy().astype(np.int64)
    assert np.array_equal(gi, oi), f"{(gi != oi).any(axis=0).sum()} signals differ"
    ynorm = np.sqrt((rows.astype(np.float64) ** 2).sum(1))[order]
    assert (np.abs(val.cpu().numpy() - ov) <= 1e-14 * ynorm + 1e-300).all()
    di, dv = _dmma_codes(eng, g, eng.m, g.perm)
    assert torch.equal(idx, di)
    assert (np.abs(val.cpu().numpy() - dv.cpu().numpy()) <= 2e-14 * ynorm + 1e-300).all()


@pytest.mark.parametrize("s0", [8, 32])
def test_residuals_match_dmma(dev, s0):
    rows = signals.patch_signals(30000, 8, 512, 512)
    eng = _engine(dev, rows, _random_blocks(4, 1), s0)
    eng.represent_full()
    g = eng.group(eng.K)
    _, _, rest, score = _ri8(eng, g, eng.m, g.perm, 1)
    r2 = torch.zeros(eng.m, dtype=torch.float64, device=dev)
    s2 = torch.zeros_like(r2)
    L.call("sbo_residual_segments", eng.sig.y.data_ptr(), eng.sig.code, 64, g.perm.data_ptr(),
           g.seg_block.data_ptr(), g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(),
           g.max_seg, eng.blocks.data_ptr(), eng.s0, eng.kind, r2.data_ptr(), s2.data_ptr(),
           eng.stream)
    torch.cuda.synchronize()
    n2 = (rows.astype(np.float64) ** 2).sum(1)
    assert (np.abs(rest.cpu().numpy() - r2.cpu().numpy()) <= 1e-13 * n2 + 1e-300).all()
    assert (np.abs(score.cpu().numpy() - s2.cpu().numpy()) <= 1e-13 * n2 + 1e-300).all()


@pytest.mark.parametrize("s0", [4, 8, 16])
def test_exact_ties_identity_block(dev, s0):
    """Q = I: c = y exactly (the digits of 1.0 are exact), and 8-bit pixel values
    repeat, so almost every signal has a magnitude tie at its threshold — every
    one goes through the exact rank rule (ties -> lower atom).  Zero signals
    (all 64 coefficients tied) keep atoms 0..k-1."""
    rows = signals.patch_signals(5000, 8, 256, 256)
    rows[::7] = 0.0
    eng = _engine(dev, rows, [np.eye(64), _random_blocks(1, 3)[0]], s0)
    g = eng.list_segments(eng.m)
    idx, val, _, _ = _ri8(eng, g, eng.m, None, 0, override=0, nblocks=2)
    oi, ov = O.top_support(rows.T.astype(np.float64), s0)
    assert np.array_equal(idx.cpu().numpy().astype(np.int64), oi)
    assert np.array_equal(val.cpu().numpy(), ov)


def test_member_list_override_and_signed_grid(dev):
    """A member list in arbitrary order coded in one block (the new block's
    rounds), negative values on the grid, all-zero signals."""
    rng = np.random.default_rng(4)
    m = 9000
    rows = (rng.integers(0, 256, (m, 64)) / 256.0 - 0.5).astype(np.float32)
    rows[rng.random(m) < 0.1] = 0.0
    blocks = _random_blocks(3, 5)
    eng = _engine(dev, rows, blocks, 8)
    members = rng.permutation(m)[:3000].astype(np.int32)
    g = eng.list_segments(3000)
    idx, val, _, _ = _ri8(eng, g, 3000, torch.from_numpy(members).to(dev), 0, override=2)
    oi, ov = _oracle_codes(rows, blocks, np.full(3000, 2), members.astype(np.int64), 8)
    assert np.array_equal(idx.cpu().numpy().astype(np.int64), oi)
    ynorm = np.sqrt((rows.astype(np.float64) ** 2).sum(1))[members]
    assert (np.abs(val.cpu().numpy() - ov) <= 1e-14 * ynorm + 1e-300).all()


def test_iteration_ri8_matches_dmma_round(dev, monkeypatch):
    """A full iteration with the digit projection equals the one with the DMMA
    projection: same decisions, blocks to 1e-11, RMSE to 1e-12."""
    from paper_1412_4944_b200.sbo import _block_rng
    rows = signals.patch_signals(1 << 16, 8, 1024, 1024)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SBO_RI8", flag)
        eng = Engine(Signals.from_rows(rows, dev), 8, k_cap=7)
        eng.set_blocks(np.stack(_random_blocks(6, 2)))
        assert eng.ri8 == (flag == "1")
        eng.represent_full()
        out = eng.iterate(4096, 6, _block_rng(0, 1, 6).standard_normal((72, 64)))
        outs.append((eng.blocks[: eng.K].cpu().numpy(), eng.state.best.cpu().numpy(),
                     eng.state.residual.cpu().numpy(), out.rmse))
    (b1, a1, r1, e1), (b0, a0, r0, e0) = outs
    assert np.array_equal(a1, a0)
    assert np.abs(b1 - b0).max() < 1e-11
    assert np.abs(r1 - r0).max() <= 1e-12 * max(r0.max(), 1e-300)
    assert abs(e1 - e0) <= 1e-12 * e0
