"""GPU parity: the CUDA path against the reference's golden outputs and the oracle.

Contract: decisions (block, support indices, worst set,
grouping) bit-exact; float64 values, energies and blocks to tight tolerances
(written per assertion).  Inputs are float32 signals (upcast for the oracle)
unless a test says otherwise.
"""
import numpy as np
import pytest
import torch

from conftest import golden
from oracle import sbo_oracle as O

pytestmark = pytest.mark.gpu

import paper_1412_4944_b200 as S  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import _block_rng  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    return require_device()


# --------------------------------------------------------------------- represent
@pytest.mark.parametrize("kind,tag", [("squared-sum", "sq"), ("abs-sum", "abs")])
def test_represent_desk_matches_reference(desk_y64, kind, tag):
    g = golden("desk_represent")
    a, code = S.represent(desk_y64, S.UnionDictionary(list(g["blocks"])), 8, kind=kind)
    np.testing.assert_array_equal(a.block, g[f"{tag}_block"])
    np.testing.assert_array_equal(code.indices, g[f"{tag}_indices"])
    np.testing.assert_allclose(code.values, g[f"{tag}_values"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(a.energy, g[f"{tag}_energy"], rtol=1e-12)
    np.testing.assert_allclose(a.residual_sq, g[f"{tag}_residual"], rtol=1e-9, atol=1e-14)


def test_represent_small_float64_signals():
    g = golden("small_cases")
    for kind, tag in (("squared-sum", "sq"), ("abs-sum", "abs")):
        a, c = S.represent(g["rep_y"], S.UnionDictionary(list(g["rep_blocks"])), 2, kind=kind)
        np.testing.assert_array_equal(a.block, g[f"rep_{tag}_block"])
        np.testing.assert_array_equal(c.indices, g[f"rep_{tag}_indices"])
        np.testing.assert_allclose(a.energy, g[f"rep_{tag}_energy"], rtol=1e-12)
        np.testing.assert_allclose(a.residual_sq, g[f"rep_{tag}_residual"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(c.values, g[f"rep_{tag}_values"], atol=1e-12)


def test_represent_gaussian_against_oracle():
    g = golden("gauss_iteration")
    from paper_1412_4944_b200 import signals
    y = signals.gaussian_signals(64, 16384, seed=5).T.astype(np.float64)
    a, c = S.represent(y, S.UnionDictionary(list(g["entering"])), 8)
    np.testing.assert_array_equal(a.block, g["rep0_block"])
    np.testing.assert_array_equal(c.indices, g["rep0_indices"])
    np.testing.assert_allclose(c.values, g["rep0_values"], atol=1e-12)
    np.testing.assert_allclose(a.residual_sq, g["rep0_residual"], rtol=1e-9, atol=1e-12)


def test_tie_prefers_lowest_block():
    rng = np.random.default_rng(5)
    q, _ = np.linalg.qr(rng.standard_normal((4, 4)))
    d = S.UnionDictionary([q, q.copy(), np.eye(4)])
    y = q @ np.array([[3.0], [0.0], [1.0], [0.0]])
    a, _ = S.represent(y, d, 2)
    assert a.block[0] == 0


def test_zero_signals_and_saturated_s0():
    rng = np.random.default_rng(2)
    qs = [np.linalg.qr(rng.standard_normal((6, 6)))[0] for _ in range(3)]
    y = np.zeros((6, 5))
    y[:, 2] = rng.standard_normal(6)
    a, c = S.represent(y, S.UnionDictionary(qs), 9)  # s0 > p keeps everything
    ra = O.code_signals(y, qs, 9)
    np.testing.assert_array_equal(a.block, ra.block)
    np.testing.assert_array_equal(c.indices, ra.indices)
    assert c.indices.shape == (6, 5)
    np.testing.assert_allclose(a.residual_sq, ra.residual_sq, atol=1e-12)


@pytest.mark.parametrize("p,K,s0,m", [(4, 3, 2, 100), (8, 5, 3, 777), (16, 4, 5, 300),
                                      (64, 16, 8, 3000), (100, 3, 12, 200), (256, 2, 16, 130)])
def test_represent_shapes_against_oracle(p, K, s0, m):
    rng = np.random.default_rng(p * 1000 + K)
    qs = [np.linalg.qr(rng.standard_normal((p, p)))[0] for _ in range(K)]
    y = rng.standard_normal((p, m))
    a, c = S.represent(y, S.UnionDictionary(qs), s0)
    r = O.code_signals(y, qs, s0)
    np.testing.assert_array_equal(a.block, r.block)
    np.testing.assert_array_equal(c.indices, r.indices)
    np.testing.assert_allclose(c.values, r.values, atol=1e-11)
    np.testing.assert_allclose(a.energy, r.energy, rtol=1e-11)


def test_represent_invariant_under_chunk_and_workers():
    rng = np.random.default_rng(13)
    qs = [np.linalg.qr(rng.standard_normal((8, 8)))[0] for _ in range(3)]
    y = np.asfortranarray(rng.standard_normal((8, 777)))
    ref = S.represent(y, S.UnionDictionary(qs), 3, chunk_size=256, workers=1)
    for chunk, workers in [(1, 1), (64, 2), (1000, 1), (300, 3)]:
        a, code = S.represent(y, S.UnionDictionary(qs), 3, chunk_size=chunk, workers=workers)
        np.testing.assert_array_equal(a.block, ref[0].block)
        np.testing.assert_array_equal(a.energy, ref[0].energy)
        np.testing.assert_array_equal(code.values, ref[1].values)


def test_represent_validation():
    rng = np.random.default_rng(3)
    d = S.UnionDictionary([np.eye(4), np.eye(4)])
    y = rng.standard_normal((4, 5))
    y[2, 3] = np.nan
    with pytest.raises(ValueError, match="NaN"):
        S.represent(y, d, 2)
    with pytest.raises(ValueError):
        S.represent(rng.standard_normal((5, 3)), d, 2)
    with pytest.raises(ValueError):
        S.represent(rng.standard_normal((4, 3)), d, 2, kind="other")


# ------------------------------------------------------------------ helpers
def test_select_top_hand_cases():
    c = S.select_top(np.array([3.0, -5.0, 1.0, 0.0]), 2)
    assert list(c.indices[:, 0]) == [0, 1] and list(c.values[:, 0]) == [3.0, -5.0]
    c = S.select_top(np.array([1.0, -1.0, 1.0]), 2)
    assert list(c.indices[:, 0]) == [0, 1] and list(c.values[:, 0]) == [1.0, -1.0]
    c = S.select_top(np.array([2.0, 0.0, -1.0]), 4)
    assert list(c.indices[:, 0]) == [0, 1, 2]
    c = S.select_top(np.array([[1.0, 4.0], [-2.0, 3.0], [0.5, -5.0]]), 2)
    assert list(c.indices[:, 1]) == [0, 2] and list(c.values[:, 1]) == [4.0, -5.0]


def test_select_top_random_against_oracle():
    rng = np.random.default_rng(9)
    for p in (1, 3, 12, 64, 130):
        c = np.round(rng.standard_normal((p, 50)), 1)  # many exact ties
        for s0 in (1, 2, 5, p + 2):
            got = S.select_top(c, s0)
            i, v = O.top_support(c, s0)
            np.testing.assert_array_equal(got.indices, i)
            np.testing.assert_array_equal(got.values, v)


def test_worst_set_cases():
    res = np.array([0.1, 0.9, 0.5])
    a = S.Assignment(np.zeros(3, np.int64), np.zeros(3), res)
    assert list(S.worst_set(a, 1)) == [1]
    a = S.Assignment(np.zeros(4, np.int64), np.zeros(4), np.full(4, 2.0))
    assert list(S.worst_set(a, 2)) == [0, 1]
    a = S.Assignment(np.zeros(3, np.int64), np.zeros(3), np.array([3.0, 1.0, 2.0]))
    assert sorted(S.worst_set(a, 10)) == [0, 1, 2]
    g = golden("small_cases")
    a = S.Assignment(np.zeros(1000, np.int64), np.zeros(1000), g["worst_res"])
    np.testing.assert_array_equal(S.worst_set(a, 100), g["worst_100"])
    rng = np.random.default_rng(4)
    r = np.round(rng.random(100000), 3)  # heavy ties at the threshold
    a = S.Assignment(np.zeros(r.size, np.int64), np.zeros(r.size), r)
    for w in (1, 77, 4096, 99999):
        np.testing.assert_array_equal(S.worst_set(a, w), O.worst_members(r, w))
    with pytest.raises(ValueError):
        S.worst_set(a, 0)


def test_group_by_block_cases():
    y = np.arange(8.0).reshape(2, 4)
    a = S.Assignment(np.array([1, 0, 1, 0]), np.zeros(4), np.zeros(4))
    grouped, ranges, perm = S.group_by_block(y, a, 2)
    assert list(perm) == [1, 3, 0, 2] and ranges == [(0, 2), (2, 4)]
    np.testing.assert_array_equal(grouped, y[:, [1, 3, 0, 2]])
    rng = np.random.default_rng(31)
    y = rng.standard_normal((5, 100000))
    blocks = rng.integers(0, 37, size=100000)
    a = S.Assignment(blocks, np.zeros(blocks.size), np.zeros(blocks.size))
    grouped, ranges, perm = S.group_by_block(y, a, 40)
    rperm, rranges = O.group_order(blocks, 40)
    np.testing.assert_array_equal(perm, rperm)
    assert ranges == rranges
    np.testing.assert_array_equal(grouped, y[:, perm])


def test_polar_and_svd_against_reference():
    g = golden("small_cases")
    np.testing.assert_allclose(S.procrustes_polar(g["polar_p8"]), g["polar_q8"], atol=1e-12)
    np.testing.assert_allclose(S.procrustes_polar(g["polar_p64"]), g["polar_q64"], atol=1e-12)
    res = S.thin_svd(g["polar_p64"])
    np.testing.assert_allclose(res.sigma, g["svd64_s"], rtol=1e-12)
    np.testing.assert_allclose(res.u, g["svd64_u"], atol=1e-10)
    np.testing.assert_allclose(res.v, g["svd64_v"], atol=1e-10)
    for shape in [(5, 3), (3, 5), (1, 1), (7, 7)]:
        a = np.random.default_rng(7).standard_normal(shape)
        r = S.thin_svd(a)
        u, s, v = O.svd(a)
        np.testing.assert_allclose(r.sigma, s, rtol=1e-12)
        np.testing.assert_allclose(r.u @ np.diag(r.sigma) @ r.v.T, a, atol=1e-12)
        np.testing.assert_allclose(r.u, u, atol=1e-10)
    assert np.allclose(S.thin_svd(np.array([[0.0, 2.0], [1.0, 0.0]])).sigma, [2.0, 1.0])
    assert np.allclose(S.procrustes_polar(np.diag([3.0, 2.0])), np.eye(2))


def test_init_onb_against_reference():
    g = golden("small_cases")
    np.testing.assert_allclose(S.init_onb(g["init_wide_y"]), g["init_wide_q"], atol=1e-10)
    np.testing.assert_allclose(S.init_onb(g["init_few_y"], np.random.default_rng(0)),
                               g["init_few_q"], atol=1e-10)
    np.testing.assert_allclose(S.init_onb(g["init_rank1_y"], np.random.default_rng(1)),
                               g["init_rank1_q"], atol=1e-10)
    np.testing.assert_allclose(S.init_onb(np.zeros((5, 7)), np.random.default_rng(2)),
                               g["init_zero_q"], atol=1e-12)
    np.testing.assert_allclose(S.init_onb(np.eye(4)), np.eye(4), atol=1e-12)
    # the caller's generator advances exactly like the reference's
    r1, r2 = np.random.default_rng(5), np.random.default_rng(5)
    S.init_onb(g["init_few_y"], r1)
    O.init_block(g["init_few_y"], r2)
    assert r1.random() == r2.random()


def test_train_onb_against_reference():
    g = golden("small_cases")
    q, c = S.train_onb(g["tr_y"], g["tr_q0"], 3, 6)
    np.testing.assert_allclose(q, g["tr_q"], atol=1e-11)
    np.testing.assert_array_equal(c.indices, g["tr_indices"])
    np.testing.assert_allclose(c.values, g["tr_values"], atol=1e-11)
    q0, code0 = S.train_onb(g["tr_y"], g["tr_q0"], 3, 0)
    np.testing.assert_array_equal(q0, g["tr_q0"])
    q, c = S.train_onb(np.empty((4, 0)), np.eye(4), 2, 3)
    assert c.num_columns == 0
    with pytest.raises(ValueError):
        S.train_onb(np.ones((4, 3)), np.eye(5), 2, 1)
    with pytest.raises(S.NumericalError):
        S.train_onb(np.ones((4, 3)), 2 * np.eye(4), 2, 1)


def test_sparse_outer_and_frobenius():
    rng = np.random.default_rng(47)
    q0 = np.linalg.qr(rng.standard_normal((7, 7)))[0]
    y = rng.standard_normal((7, 60))
    i, v = O.top_support(q0.T @ y, 3)
    code = S.ThresholdedCode(i, v)
    np.testing.assert_allclose(S.sparse_outer(y, code), O.outer_sparse(y, i, v), atol=1e-12)
    e = S.frobenius_error(y, q0, code)
    assert e == pytest.approx(np.linalg.norm(y - q0 @ code.to_csc(7).toarray()), rel=1e-12)


# ------------------------------------------------------------- the iteration
def _engine(dev, y32, blocks, s0=8):
    eng = Engine(Signals.from_rows(y32, dev), s0, k_cap=len(blocks) + 1)
    eng.set_blocks(np.stack(blocks))
    eng.represent_full()
    return eng


def test_iteration_desk_teacher_forced(dev, desk_y32):
    """Desk iteration.  Its new block's first Procrustes matrix has two exactly-zero
    columns (atoms no worst-set signal selects), so the reference's block there is
    LAPACK's arbitrary null-space completion: the new block is teacher-forced and
    everything downstream (represent #1, grouping, retraining, represent #2) must
    match; the new block's own pieces are checked separately below."""
    g = golden("desk_iteration")
    eng = _engine(dev, desk_y32, list(g["entering"]))
    np.testing.assert_allclose(eng.state.residual.cpu().numpy(), g["entering_residual"],
                               rtol=1e-9, atol=1e-14)
    K = eng.K
    out = eng.iterate(512, 6, None, force_new_block=g["new_block_rounds"][-1])
    np.testing.assert_array_equal(np.sort(out.worst.cpu().numpy()), np.sort(g["worst"]))
    blocks = eng.blocks[: eng.K].cpu().numpy()
    err = max(np.abs(blocks[b] - g["retrained"][b]).max() for b in range(K + 1))
    assert err < 1e-9, err
    np.testing.assert_array_equal(eng.state.best.cpu().numpy(), g["rep2_block"])
    np.testing.assert_allclose(eng.state.residual.cpu().numpy(), g["rep2_residual"],
                               rtol=1e-8, atol=1e-13)
    assert out.rmse == pytest.approx(float(g["rmse"]), rel=1e-10)


def test_desk_new_block_init_and_degenerate_polar(dev, desk_y32):
    """The new block's init (Gram + Jacobi) matches gesdd's U; on the rank-deficient
    first round our polar factor is an equally optimal Procrustes solution."""
    g = golden("desk_iteration")
    y64 = desk_y32.T.astype(np.float64)
    ysub = y64[:, g["worst"]]
    q0 = S.init_onb(ysub, _block_rng(1, 1, 4))
    np.testing.assert_allclose(q0, g["init_block"], atol=1e-8)
    i, v = O.top_support(g["init_block"].T @ ysub, 8)
    P = O.outer_sparse(ysub, i, v)
    assert (np.abs(P).sum(axis=0) == 0).sum() == 2
    q = S.procrustes_polar(P)
    assert S.orthonormality_defect(q) <= 1e-12
    u, s, vt = np.linalg.svd(P)
    assert np.trace(q.T @ P) == pytest.approx(s.sum(), rel=1e-12)
    r = int((s > s[0] * 1e-9).sum())  # on the range of P^T both factors agree
    np.testing.assert_allclose(q @ vt[:r].T, u[:, :r], atol=1e-6)


def test_iteration_gaussian_teacher_forced(dev):
    from paper_1412_4944_b200 import signals
    g = golden("gauss_iteration")
    y32 = signals.gaussian_signals(64, 16384, seed=5)
    eng = _engine(dev, y32, list(g["entering"]))
    K = eng.K
    draws = _block_rng(0, 1, K).standard_normal((64 + 8, 64))
    out = eng.iterate(1024, 6, draws)
    np.testing.assert_array_equal(np.sort(out.worst.cpu().numpy()), np.sort(g["worst"]))
    blocks = eng.blocks[: eng.K].cpu().numpy()
    assert np.abs(blocks - g["retrained"]).max() < 1e-9
    np.testing.assert_array_equal(eng.state.best.cpu().numpy(), g["rep2_block"])


def test_sbo_init_desk(desk_y64):
    g = golden("desk_represent")
    d = S.sbo_init(desk_y64, S.SboConfig(s0=8, k0=4, p0=4096, rounds=6, seed=1))
    for q, r in zip(d.blocks, g["blocks"]):
        np.testing.assert_allclose(q, r, atol=1e-10)


def test_sbo_train_config_a(desk_y64):
    g = golden("desk_train")
    d, code, a, rep = S.sbo_train(desk_y64, S.SboConfig(s0=8, k0=4, p0=4096, rounds=6,
                                                        k_max=14, seed=0))
    rm = np.array([r.rmse for r in rep.rows])
    assert d.num_blocks == 14 and len(rep.rows) == 11
    np.testing.assert_allclose(rm, g["rmse"], rtol=1e-3)  # chaotic trajectory
    assert all(b <= a * (1 + 1e-12) for a, b in zip(rm, rm[1:]))
    assert rep.rmse_recomputed == pytest.approx(rep.rmse_final, abs=1e-10)
    for q in d.blocks:
        assert S.orthonormality_defect(q) <= 1e-8


def test_sbo_train_contracts():
    rng = np.random.default_rng(67)
    y = rng.standard_normal((6, 300))
    d, code, a, rep = S.sbo_train(y, S.SboConfig(s0=2, k0=5, p0=64, k_max=8, seed=7, rounds=2))
    assert d.num_blocks == 8 and [r.dictionary_size for r in rep.rows] == [5, 6, 7, 8]
    _, _, rmses, _ = O.train(y, 2, k0=5, p0=64, rounds=2, k_max=8, seed=7)
    np.testing.assert_allclose([r.rmse for r in rep.rows], rmses, rtol=1e-10)
    for kind in ("squared-sum", "abs-sum"):
        y = np.random.default_rng(89).standard_normal((6, 200))
        d, _, _, rep = S.sbo_train(y, S.SboConfig(s0=2, k0=2, p0=50, k_max=4, seed=23, rounds=2,
                                                  energy_kind=kind))
        blocks, rep_o, rmses, _ = O.train(y, 2, k0=2, p0=50, rounds=2, k_max=4, seed=23,
                                          kind=kind)
        np.testing.assert_allclose([r.rmse for r in rep.rows], rmses, rtol=1e-10)


def test_empty_block_left_unchanged_and_noted(dev):
    """A duplicated block loses every tie to its twin (lowest index wins), so it
    serves no signal: it must be left unchanged and reported (sbo.py:379-383)."""
    from paper_1412_4944_b200.report import TrainReport
    from paper_1412_4944_b200.sbo import SboConfig, train_engine
    rng = np.random.default_rng(3)
    p, m = 8, 2000
    y32 = rng.standard_normal((m, p)).astype(np.float32)
    q0, q1 = (np.linalg.qr(rng.standard_normal((p, p)))[0] for _ in range(2))
    entering = [q0, q1, q0.copy()]
    eng = _engine(dev, y32, entering, s0=3)
    out = eng.iterate(max(p, m // 16), 3, _block_rng(0, 1, 3).standard_normal((p + 8, p)))
    y64 = y32.T.astype(np.float64)
    rep0 = O.code_signals(y64, entering, 3)
    tr = O.iterate(y64, entering, rep0.residual_sq, 3, 3, max(p, m // 16), seed=0)
    assert out.empty_blocks == tr.empty == [2]
    np.testing.assert_array_equal(eng.blocks[2].cpu().numpy(), q0)
    for a, b in zip(eng.blocks[: eng.K].cpu().numpy(), tr.blocks):
        np.testing.assert_allclose(a, b, atol=1e-10)
    eng = _engine(dev, y32, entering, s0=3)
    rep = TrainReport("sbo", {}, 0, 1)
    train_engine(eng, SboConfig(s0=3, k0=3, k_max=4, rounds=3, seed=0), max(p, m // 16), rep)
    assert rep.notes == ["iteration 1: block 2 had no signals, left unchanged"]


def test_sbo_train_fixed_point():
    rng = np.random.default_rng(61)
    q_star = np.linalg.qr(rng.standard_normal((5, 5)))[0]
    x = np.zeros((5, 40))
    for j in range(40):
        x[j % 5, j] = 5.0 - (j % 5) * 0.9 + 0.01 * (j // 5)
    d, code, a, rep = S.sbo_train(q_star @ x, S.SboConfig(s0=1, k0=1, p0=40, k_max=8,
                                                         target_error=1e-8, seed=5, rounds=4))
    assert d.num_blocks == 1 and rep.rows[-1].rmse <= 1e-8


@pytest.mark.parametrize("s0", [8, 16])
def test_iteration_zero_and_duplicate_signals(dev, s0):
    """Multi-tile segments mixing all-zero signals (every coefficient ties at 0: the
    exact rank fallback, index order), small duplicated signals (scaled below the
    worst set, which would otherwise be rank-deficient) and Gaussian ones:
    represent, the fused rounds and the residual pass vs the oracle."""
    rng = np.random.default_rng(21)
    p, m, K = 64, 24576, 4
    y32 = rng.standard_normal((m, p)).astype(np.float32)
    y32[rng.random(m) < 0.2] = 0.0
    dup = rng.random(m) < 0.2
    y32[dup] = 0.05 * y32[np.flatnonzero(~dup)[:7]][rng.integers(0, 7, dup.sum())]
    blocks = [np.linalg.qr(rng.standard_normal((p, p)))[0] for _ in range(K)]
    eng = _engine(dev, y32, blocks, s0)
    y64 = y32.T.astype(np.float64)
    rep0 = O.code_signals(y64, blocks, s0)
    np.testing.assert_array_equal(eng.state.best.cpu().numpy(), rep0.block)
    np.testing.assert_allclose(eng.state.residual.cpu().numpy(), rep0.residual_sq,
                               rtol=1e-9, atol=1e-12)
    draws = _block_rng(0, 1, K).standard_normal((p + 8, p))
    out = eng.iterate(m // 16, 3, draws)
    tr = O.iterate(y64, blocks, rep0.residual_sq, s0, 3, m // 16, seed=0)
    np.testing.assert_array_equal(np.sort(out.worst.cpu().numpy()), np.sort(tr.worst))
    got = eng.blocks[: eng.K].cpu().numpy()
    assert max(np.abs(a - b).max() for a, b in zip(got, tr.blocks)) < 1e-9
    np.testing.assert_array_equal(eng.state.best.cpu().numpy(), tr.rep2.block)
    np.testing.assert_allclose(eng.state.residual.cpu().numpy(), tr.rep2.residual_sq,
                               rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("p,K,s0,m", [(64, 3, 16, 6000), (64, 3, 32, 4000), (16, 4, 4, 5000),
                                      (256, 2, 16, 32768)])
def test_iteration_other_shapes_against_oracle(dev, p, K, s0, m):
    """Configs D/E shapes (p = 256, s0 in {16, 32}) and a small p: the general float64
    path (no fused round) through one full teacher-free iteration vs the oracle."""
    rng = np.random.default_rng(1000 * p + s0)
    y32 = rng.standard_normal((m, p)).astype(np.float32)
    blocks = [np.linalg.qr(rng.standard_normal((p, p)))[0] for _ in range(K)]
    eng = _engine(dev, y32, blocks, s0)
    y64 = y32.T.astype(np.float64)
    rep0 = O.code_signals(y64, blocks, s0)
    np.testing.assert_array_equal(eng.state.best.cpu().numpy(), rep0.block)
    w = max(p, m // 16)
    draws = _block_rng(0, 1, K).standard_normal((p + 8, p))
    out = eng.iterate(w, 2, draws)
    tr = O.iterate(y64, blocks, rep0.residual_sq, s0, 2, w, seed=0)
    np.testing.assert_array_equal(np.sort(out.worst.cpu().numpy()), np.sort(tr.worst))
    got = eng.blocks[: eng.K].cpu().numpy()
    assert max(np.abs(a - b).max() for a, b in zip(got, tr.blocks)) < 1e-8
    np.testing.assert_array_equal(eng.state.best.cpu().numpy(), tr.rep2.block)
    np.testing.assert_allclose(eng.state.residual.cpu().numpy(), tr.rep2.residual_sq,
                               rtol=1e-9, atol=1e-12)
    assert out.rmse == pytest.approx(tr.rmse, rel=1e-10)


def test_graph_replayed_iteration_matches_eager(dev):
    """The bench's CUDA-graph step (restore + Engine.iterate_device) gives the same
    blocks, assignment, residuals and RMSE as an eager iteration, on every replay."""
    from paper_1412_4944_b200 import signals
    g = golden("gauss_iteration")
    y32 = signals.gaussian_signals(64, 16384, seed=5)
    eng = _engine(dev, y32, list(g["entering"]))
    K = eng.K
    snap = eng.snapshot()
    draws = _block_rng(0, 1, K).standard_normal((64 + 8, 64))
    ref = eng.iterate(1024, 6, draws)
    want = (eng.blocks[: eng.K].cpu().numpy(), eng.state.best.cpu().numpy(),
            eng.state.residual.cpu().numpy())
    replay = eng.capture_iteration(snap, 1024, 6, torch.from_numpy(draws).to(dev))
    for _ in range(2):
        out = replay()
        np.testing.assert_array_equal(eng.blocks[: eng.K].cpu().numpy(), want[0])
        np.testing.assert_array_equal(eng.state.best.cpu().numpy(), want[1])
        np.testing.assert_array_equal(eng.state.residual.cpu().numpy(), want[2])
        assert out.rmse == ref.rmse and out.K == ref.K


def test_p0_above_m_samples_with_replacement():
    """Reference test_sbo.py:272-280 (sbo.py:275-280, 326-329): p0 > m samples
    the start-up columns with replacement — sbo_init warns, sbo_train notes it
    in the report instead (it silences sbo_init's warning) — and the trajectory
    equals the oracle's (which draws the same columns)."""
    import warnings
    y = np.random.default_rng(31).standard_normal((6, 40))
    cfg = S.SboConfig(s0=2, k0=2, p0=100, k_max=3, seed=11, rounds=2)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        d, _, _, rep = S.sbo_train(y, cfg)
    assert any("replacement" in n for n in rep.notes)
    blocks, _, rmses, _ = O.train(y, 2, k0=2, p0=100, rounds=2, k_max=3, seed=11)
    np.testing.assert_allclose([r.rmse for r in rep.rows], rmses, rtol=1e-10)
    with pytest.warns(UserWarning, match="replacement"):
        d0 = S.sbo_init(y, cfg)
    for q in d0.blocks:
        assert S.orthonormality_defect(q) <= 1e-8
