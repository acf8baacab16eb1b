"""The p = 256 projection on tcgen05 from exact integer digits (coef_i8.cu;
onb.py:170 Q^T Y) and the selection on its rows (sbo_select_coded), against
the CPU oracle and the float64 DMMA coding kernel (sbo_code_segments) on the
same signals and blocks.

Contract: coefficients within 1e-15 of ||y||_1 of the exact float64 product
(Q is rounded to 2^-54, dropped digit levels weigh <= 2^-49 relative);
supports bit-exact (ties -> lower atom, oracle.top_support); values to 1e-14
of ||y||; residuals / scores to 1e-13 of ||y||^2."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import sbo_oracle as O  # noqa: E402
from paper_1412_4944_b200 import _lib as L  # noqa: E402
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402

P = 256


@pytest.fixture(scope="module")
def dev():
    return require_device()


@pytest.fixture(autouse=True)
def _ci8_on(monkeypatch):
    monkeypatch.setenv("SBO_I8", "1")
    monkeypatch.setenv("SBO_CI8", "1")


def _blocks(K, seed):
    rng = np.random.default_rng(seed)
    return [np.linalg.qr(rng.standard_normal((P, P)))[0] for _ in range(K)]


def _engine(dev, rows, blocks, s0):
    eng = Engine(Signals.from_rows(rows, dev), s0, k_cap=len(blocks))
    eng.set_blocks(np.stack(blocks))
    assert eng.ci8 and eng.ysy is not None
    return eng


def _coef(eng, g, n, order, override=-1, nblocks=None):
    nb = nblocks or eng.K
    ws = torch.empty(L.size("sbo_coef_i8_workspace_bytes", nb), dtype=torch.uint8,
                     device=eng.dev)
    coef = torch.full((max(n, 1), P), np.nan, dtype=torch.float64, device=eng.dev)
    L.call("sbo_coef_i8_segments", eng.ydig.data_ptr(), eng.ysy,
           order.data_ptr() if order is not None else None, g.seg_block.data_ptr(),
           g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg,
           eng.blocks.data_ptr(), nb, override, coef.data_ptr(), ws.data_ptr(), ws.numel(),
           eng.stream)
    torch.cuda.synchronize()
    return coef


def _block_of_positions(g, n):
    lo, hi = g.seg_lo.cpu().numpy(), g.seg_hi.cpu().numpy()
    sb = g.seg_block.cpu().numpy()
    out = np.full(n, -1, np.int64)
    for s in range(int(g.nseg.item())):
        out[lo[s]:hi[s]] = sb[s]
    return out


def _exact_coef(rows, blocks, block_of_pos, order):
    y = rows.astype(np.float64)[order]
    c = np.empty((len(order), P))
    for b in np.unique(block_of_pos):
        sel = np.nonzero(block_of_pos == b)[0]
        c[sel] = y[sel] @ blocks[b]
    return c


def test_coefficients_grouped(dev):
    """Unit-range 16x16 patches, 5 blocks, the representation's grouping
    (ragged per-block tails, many segments)."""
    rows = signals.patch_signals(6000 + 77, 16, 512, 512)
    blocks = _blocks(5, 1)
    eng = _engine(dev, rows, blocks, 8)
    eng.represent_full()
    g = eng.group(eng.K)
    c = _coef(eng, g, eng.m, g.perm).cpu().numpy()
    order = g.perm.cpu().numpy().astype(np.int64)
    ref = _exact_coef(rows, blocks, _block_of_positions(g, eng.m), order)
    l1 = np.abs(rows.astype(np.float64)).sum(1)[order]
    assert (np.abs(c - ref) <= 1e-15 * l1[:, None] + 1e-300).all()


def test_coefficients_signed_override_zero_rows(dev):
    """A member list in arbitrary order coded in one block, signed values on
    the grid, all-zero signals (coefficients exactly 0)."""
    rng = np.random.default_rng(4)
    m = 3000
    rows = (rng.integers(0, 256, (m, P)) / 256.0 - 0.5).astype(np.float32)
    rows[rng.random(m) < 0.1] = 0.0
    blocks = _blocks(3, 5)
    eng = _engine(dev, rows, blocks, 8)
    members = rng.permutation(m)[:1000].astype(np.int32)
    g = eng.list_segments(1000)
    c = _coef(eng, g, 1000, torch.from_numpy(members).to(dev), override=2).cpu().numpy()
    ref = _exact_coef(rows, blocks, np.full(1000, 2), members.astype(np.int64))
    l1 = np.abs(rows.astype(np.float64)).sum(1)[members]
    assert (np.abs(c - ref) <= 1e-15 * l1[:, None] + 1e-300).all()
    zero = ~rows[members].any(axis=1)
    assert zero.any() and (c[zero] == 0).all()


def test_identity_block_is_exact(dev):
    """Q = I: every digit of 1.0 and 0.0 is exact, so C = Y bit for bit."""
    rows = signals.patch_signals(2000, 16, 256, 256)
    eng = _engine(dev, rows, [np.eye(P)], 4)
    g = eng.list_segments(eng.m)
    c = _coef(eng, g, eng.m, None, override=0).cpu().numpy()
    assert np.array_equal(c, rows.astype(np.float64))


@pytest.mark.parametrize("s0", [4, 16, 64])
def test_select_coded_matches_oracle_and_dmma(dev, s0):
    rows = signals.patch_signals(5000, 16, 512, 512)
    blocks = _blocks(4, s0)
    eng = _engine(dev, rows, blocks, s0)
    eng.represent_full()
    g = eng.group(eng.K)
    n, k, ld = eng.m, eng.k, eng.m
    idx = torch.full((k, ld), -7, dtype=torch.int16, device=dev)
    val = torch.full((k, ld), np.nan, dtype=torch.float64, device=dev)
    eng.code_i8(g.perm, g, n, eng.K, -1, ld, idx, val)
    torch.cuda.synchronize()
    order = g.perm.cpu().numpy().astype(np.int64)
    bop = _block_of_positions(g, n)
    oi = np.empty((k, n), np.int64)
    ov = np.empty((k, n))
    y = rows.astype(np.float64)[order]
    for b in np.unique(bop):
        sel = np.nonzero(bop == b)[0]
        oi[:, sel], ov[:, sel] = O.top_support(blocks[b].T @ y[sel].T, s0)
    gi = idx.cpu().numpy().astype(np.int64)
    assert np.array_equal(gi, oi), f"{(gi != oi).any(axis=0).sum()} signals differ"
    ynorm = np.sqrt((y ** 2).sum(1))
    assert (np.abs(val.cpu().numpy() - ov) <= 1e-14 * ynorm + 1e-300).all()
    di = torch.zeros_like(idx)
    dv = torch.zeros_like(val)
    eng.code(g.perm, g, -1, False, ld, di, dv)
    torch.cuda.synchronize()
    assert torch.equal(idx, di)
    assert (np.abs(val.cpu().numpy() - dv.cpu().numpy()) <= 2e-14 * ynorm + 1e-300).all()


def test_select_coded_residuals_by_signal(dev):
    rows = signals.patch_signals(4000, 16, 512, 512)
    eng = _engine(dev, rows, _blocks(3, 9), 16)
    eng.represent_full()
    g = eng.group(eng.K)
    r1 = torch.full((eng.m,), np.nan, dtype=torch.float64, device=dev)
    s1 = torch.full_like(r1, np.nan)
    eng.code_i8(g.perm, g, eng.m, eng.K, -1, eng.m, None, None, s1, r1, by_signal=True)
    r2 = torch.zeros_like(r1)
    s2 = torch.zeros_like(r1)
    eng.code(g.perm, g, -1, True, eng.m, None, None, s2, r2)
    torch.cuda.synchronize()
    n2 = (rows.astype(np.float64) ** 2).sum(1)
    assert (np.abs(r1.cpu().numpy() - r2.cpu().numpy()) <= 1e-13 * n2 + 1e-300).all()
    assert (np.abs(s1.cpu().numpy() - s2.cpu().numpy()) <= 1e-13 * n2 + 1e-300).all()


def test_iteration_ci8_matches_dmma(dev, monkeypatch):
    """A full p = 256 iteration with the digit projection equals the one with the
    DMMA projection: same decisions, blocks to 1e-11, RMSE to 1e-12."""
    from paper_1412_4944_b200.sbo import _block_rng
    rows = signals.patch_signals(1 << 14, 16, 1024, 1024)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SBO_CI8", flag)
        eng = Engine(Signals.from_rows(rows, dev), 8, k_cap=5)
        eng.set_blocks(np.stack(_blocks(4, 2)))
        assert eng.ci8 == (flag == "1")
        eng.represent_full()
        out = eng.iterate(1024, 4, _block_rng(0, 1, 4).standard_normal((P + 8, P)))
        outs.append((eng.blocks[: eng.K].cpu().numpy(), eng.state.best.cpu().numpy(),
                     eng.state.residual.cpu().numpy(), out.rmse))
    (b1, a1, r1, e1), (b0, a0, r0, e0) = outs
    assert np.array_equal(a1, a0)
    assert np.abs(b1 - b0).max() < 1e-11
    assert np.abs(r1 - r0).max() <= 1e-12 * max(r0.max(), 1e-300)
    assert abs(e1 - e0) <= 1e-12 * e0


@pytest.mark.parametrize("kind", ["squared-sum", "abs-sum"])
def test_recheck_i8_near_tied_blocks_match_oracle(dev, kind, monkeypatch):
    """Perturbed copies of the signals' principal basis: every signal's
    energies are within the tensor-core certificate in several blocks, so most
    signals go to the float64 re-decision with multi-block candidate masks.
    Decisions equal the oracle's through the pair lists
    (sbo_energy_recheck_pairs), the tile unions (sbo_energy_recheck_i8) and the
    DMMA recheck; the two digit rechecks agree bit for bit."""
    rows = signals.patch_signals(3000, 16, 512, 512)
    # only near-copies compete
    base = np.linalg.eigh(rows.T.astype(np.float64) @ rows.astype(np.float64))[1][:, ::-1]
    qs = [np.ascontiguousarray(base)]
    rng = np.random.default_rng(21)
    for i in range(5):  # perturbed copies: energies 1e-8 .. 1e-7 apart, no exact ties
        q, r = np.linalg.qr(base + 2e-8 * (i + 1) * rng.standard_normal((P, P)))
        qs.append(q * np.sign(np.diag(r)))
    states = []
    for flag, pairs in (("1", "1"), ("1", "0"), ("0", "1")):
        monkeypatch.setenv("SBO_CI8", flag)
        monkeypatch.setenv("SBO_RECHECK_PAIRS", pairs)
        eng = Engine(Signals.from_rows(rows, dev), 16, kind, k_cap=len(qs))
        eng.set_blocks(np.stack(qs))
        assert eng.ci8 == (flag == "1")
        eng.energy(0, eng.K, False)
        torch.cuda.synchronize()
        assert int(eng.nflag.item()) > 1000  # the re-decision is exercised
        st = eng.state
        states.append((st.best.cpu().numpy(), st.score.cpu().numpy(),
                       st.residual.cpu().numpy()))
    r = O.code_signals(rows.T.astype(np.float64), qs, 16, kind)
    (bp, sp, rp), (b1, s1, r1), (b0, s0_, r0) = states  # pairs, tile unions, DMMA
    np.testing.assert_array_equal(bp, r.block)
    np.testing.assert_array_equal(b1, r.block)
    np.testing.assert_array_equal(b0, r.block)
    assert np.array_equal(sp, s1) and np.array_equal(rp, r1)  # same digits, same selection
    n2 = (rows.astype(np.float64) ** 2).sum(1)
    assert (np.abs(s1 - s0_) <= 1e-13 * n2 + 1e-300).all()
    assert (np.abs(r1 - r0) <= 1e-13 * n2 + 1e-300).all()


@pytest.mark.parametrize("s0", [1, 16, 32])
def test_code_i8_exact_ties_identity_block(dev, s0):
    """Q = I: the coefficients are the 8-bit pixel values, so nearly every signal
    has magnitude ties at its threshold (and zero signals tie everywhere): the
    exact rank rule (ties -> lower atom) must match oracle.top_support."""
    rows = signals.patch_signals(4000, 16, 256, 256)
    rows[::9] = 0.0
    eng = _engine(dev, rows, [np.eye(P), _blocks(1, 3)[0]], s0)
    g = eng.list_segments(eng.m)
    n, k = eng.m, eng.k
    idx = torch.full((k, n), -7, dtype=torch.int16, device=dev)
    val = torch.full((k, n), np.nan, dtype=torch.float64, device=dev)
    eng.code_i8(None, g, n, 2, 0, n, idx, val)
    torch.cuda.synchronize()
    oi, ov = O.top_support(rows.T.astype(np.float64), s0)
    assert np.array_equal(idx.cpu().numpy().astype(np.int64), oi)
    assert np.array_equal(val.cpu().numpy(), ov)
