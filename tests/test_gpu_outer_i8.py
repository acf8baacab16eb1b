"""The tensor-core outer product P = Y X^T (outer_i8.cu, onb.py:127-134) against the
float64 kernels on identical codes, and the coding half of the round
(sbo_round_code_segments) against sbo_code_segments.

Contract: codes (indices) bit-exact, code values to 1e-13 relative (float64
projections in a different summation order); partials P to 1e-13 of max |P|
(the integer-digit product is exact up to the 2^-sx rounding of the code values
and the dropped digit levels, far below float64 summation error)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1412_4944_b200 import _lib as L  # noqa: E402
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    return require_device()


@pytest.fixture(autouse=True)
def _i8_on(monkeypatch):
    monkeypatch.setenv("SBO_I8", "1")


def _setup(dev, rows, K, s0, seed=0):
    rng = np.random.default_rng(seed)
    eng = Engine(Signals.from_rows(rows, dev), s0, k_cap=K)
    eng.set_blocks(np.stack([np.linalg.qr(rng.standard_normal((64, 64)))[0] for _ in range(K)]))
    eng.represent_full()
    return eng


def _p_i8_and_f64(eng, g, n, order, nblocks, idx, val, seg_block):
    """P per block from the tensor-core kernel, and from the float64 outer product
    + ordered reduction, on the same codes."""
    st, ld = eng.stream, max(n, 1)
    order_p = order.data_ptr() if order is not None else None
    P_i8 = torch.zeros((nblocks, 64, 64), dtype=torch.float64, device=eng.dev)
    P_f64 = torch.zeros_like(P_i8)
    ws = torch.empty(L.size("sbo_outer_i8_workspace_bytes", nblocks, 64), dtype=torch.uint8,
                     device=eng.dev)
    sy, sx = eng.i8
    tiles = torch.empty(L.size("sbo_y_tiles_bytes", n, g.max_seg, 64), dtype=torch.uint8,
                        device=eng.dev)
    L.call("sbo_y_tiles", eng.ydig.data_ptr(), 64, order_p, g.seg_lo.data_ptr(), g.seg_hi.data_ptr(),
           g.nseg.data_ptr(), g.max_seg, tiles.data_ptr(), st)
    L.call("sbo_outer_i8_segments", tiles.data_ptr(), 64,
           seg_block.data_ptr() if seg_block is not None else None, g.seg_lo.data_ptr(),
           g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg, nblocks, eng.s0, ld,
           idx.data_ptr(), val.data_ptr(), sy, sx, P_i8.data_ptr(), ws.data_ptr(), ws.numel(), st)
    part = torch.zeros((g.max_seg, 64, 64), dtype=torch.float64, device=eng.dev)
    L.call("sbo_outer_segments", eng.sig.y.data_ptr(), eng.sig.code, 64, order_p,
           g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg, eng.s0, ld,
           idx.data_ptr(), val.data_ptr(), part.data_ptr(), st)
    L.call("sbo_reduce_segments", part.data_ptr(),
           seg_block.data_ptr() if seg_block is not None else None, g.nseg.data_ptr(),
           g.max_seg, nblocks, 64, P_f64.data_ptr(), st)
    torch.cuda.synchronize()
    return P_i8.cpu().numpy(), P_f64.cpu().numpy()


def _codes(eng, g, n, order, override=-1):
    k, ld, st = eng.k, max(n, 1), eng.stream
    y = eng.sig.y.data_ptr()
    mk = lambda dt: torch.zeros((k, ld), dtype=dt, device=eng.dev)  # noqa: E731
    idx_a, val_a, idx_b, val_b = mk(torch.int16), mk(torch.float64), mk(torch.int16), mk(torch.float64)
    common = (g.seg_block.data_ptr(), g.seg_lo.data_ptr(), g.seg_hi.data_ptr(),
              g.nseg.data_ptr(), g.max_seg, eng.blocks.data_ptr(), override, eng.s0)
    order_p = order.data_ptr() if order is not None else None
    L.call("sbo_round_code_segments", y, eng.sig.code, 64, order_p, *common, ld,
           idx_a.data_ptr(), val_a.data_ptr(), st)
    L.call("sbo_code_segments", y, eng.sig.code, 64, order_p, *common, eng.kind, 0, ld,
           idx_b.data_ptr(), val_b.data_ptr(), None, None, st)
    torch.cuda.synchronize()
    return idx_a, val_a, idx_b, val_b


def _close(pi, pf):
    for b in range(pf.shape[0]):
        scale = max(np.abs(pf[b]).max(), 1e-300)
        assert np.abs(pi[b] - pf[b]).max() <= 1e-13 * scale, (b, np.abs(pi[b] - pf[b]).max())


@pytest.mark.parametrize("s0", [4, 8, 16, 32])
def test_round_codes_and_i8_products_patches(dev, s0):
    """Unit-range patches (the benchmark's format), ragged segments (the group's
    per-block tails are not multiples of the 128-signal tile)."""
    rows = signals.patch_signals(20000 + 37, 8, 512, 512)
    eng = _setup(dev, rows, 5, s0)
    assert eng.i8 is not None, "unit-range patches must take the integer-digit path"
    g = eng.group(eng.K)
    ia, va, ib, vb = _codes(eng, g, eng.m, g.perm)
    assert torch.equal(ia, ib)
    np.testing.assert_allclose(va.cpu().numpy(), vb.cpu().numpy(), rtol=1e-13, atol=1e-15)
    pi, pf = _p_i8_and_f64(eng, g, eng.m, g.perm, eng.K, ia, va, g.seg_block)
    _close(pi, pf)


def test_i8_products_signed_zero_and_member_list(dev):
    """Negative values (a signed grid: k/256 - 1/2), all-zero signals and a member
    list in arbitrary order (the new block's segments, no segment blocks)."""
    rng = np.random.default_rng(4)
    m = 9000
    rows = (rng.integers(0, 256, (m, 64)) / 256.0 - 0.5).astype(np.float32)
    rows[rng.random(m) < 0.1] = 0.0
    eng = _setup(dev, rows, 3, 8, seed=1)
    assert eng.i8 is not None
    members = torch.from_numpy(rng.permutation(m)[:3000].astype(np.int32)).to(dev)
    g = eng.list_segments(3000)
    ia, va, _, _ = _codes(eng, g, 3000, members, override=1)
    pi, pf = _p_i8_and_f64(eng, g, 3000, members, 1, ia, va, None)
    _close(pi, pf)


def test_i8_products_independent_of_segmentation(dev, monkeypatch):
    """Exact integer accumulation: the same signals cut into different segment
    tables give bit-identical P."""
    import paper_1412_4944_b200.engine as E
    rows = signals.patch_signals(30000, 8, 512, 512)
    outs = []
    for seg in (1024, 256):
        monkeypatch.setattr(E, "SEG_LEN", seg)
        eng = _setup(dev, rows, 4, 8)
        g = eng.group(eng.K)
        ia, va, _, _ = _codes(eng, g, eng.m, g.perm)
        outs.append(_p_i8_and_f64(eng, g, eng.m, g.perm, eng.K, ia, va, g.seg_block)[0])
    assert np.array_equal(outs[0], outs[1])


def test_gaussian_signals_keep_the_float64_round(dev):
    """float32 Gaussian values span more than the 35-bit grid: the engine keeps the
    fused float64 DMMA round (no integer-digit product)."""
    rows = signals.gaussian_signals(64, 4096, seed=3)
    eng = _setup(dev, rows, 2, 8)
    assert eng.i8 is None


def test_iteration_i8_matches_float64_round(dev, monkeypatch):
    """One full iteration with the integer-digit outer product equals the one with
    the fused float64 round: same decisions, blocks to 1e-11."""
    from paper_1412_4944_b200.sbo import _block_rng
    rows = signals.patch_signals(1 << 16, 8, 1024, 1024)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SBO_I8", flag)
        eng = _setup(dev, rows, 6, 8, seed=2)
        assert (eng.i8 is not None) == (flag == "1")
        out = eng.iterate(4096, 6, _block_rng(0, 1, 6).standard_normal((72, 64)))
        outs.append((eng.blocks[: eng.K].cpu().numpy(), eng.state.best.cpu().numpy(),
                     out.rmse))
    (b1, a1, r1), (b0, a0, r0) = outs
    assert np.abs(b1 - b0).max() <= 1e-11
    np.testing.assert_array_equal(a1, a0)
    assert r1 == pytest.approx(r0, rel=1e-12)
