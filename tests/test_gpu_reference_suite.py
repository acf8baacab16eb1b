"""The reference's own hot-path test strategy (tests/test_onb.py,
test_sbo.py, test_linalg.py, test_acceptance.py 1-6/9/11), restated against this
package on the GPU: hand cases, brute-force oracles and invariants.  Each test
names the reference test it mirrors."""
import itertools

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st
from hypothesis.extra import numpy as nph

pytestmark = pytest.mark.gpu

import paper_1412_4944_b200 as S  # noqa: E402
from paper_1412_4944_b200 import data, signals, store  # noqa: E402


def orth(p, rng):
    q, _ = np.linalg.qr(rng.standard_normal((p, p)))
    return q


def canonical(q):
    piv = np.argmax(np.abs(q), axis=0)
    return q * np.where(q[piv, np.arange(q.shape[1])] < 0, -1.0, 1.0)


# ---------------------------------------------------------------- select_top
@settings(max_examples=60, deadline=None)
@given(nph.arrays(np.float64, st.integers(1, 12), elements=st.floats(-1e6, 1e6, allow_nan=False)),
       st.integers(1, 14))
def test_select_top_brute_force(x, s0):  # test_onb.py:61
    code = S.select_top(x, s0)
    k = min(s0, x.shape[0])
    assert code.indices.shape == (k, 1)
    assert np.all(np.diff(code.indices[:, 0]) > 0)
    want = sorted(range(x.shape[0]), key=lambda i: (-abs(x[i]), i))[:k]
    assert set(code.indices[:, 0]) == set(want)
    np.testing.assert_array_equal(code.values[:, 0], x[code.indices[:, 0]])


def test_select_top_coding_optimality():  # test_onb.py:71, acceptance 05
    rng = np.random.default_rng(99)
    p = 6
    for s0 in (1, 2, 3):
        for _ in range(10):
            q = orth(p, rng)
            y = rng.standard_normal(p)
            c = q.T @ y
            code = S.select_top(c, s0)
            got = np.sum(y ** 2) - np.sum(code.values[:, 0] ** 2)
            best = min(np.sum(y ** 2) - np.sum(c[list(sup)] ** 2)
                       for sup in itertools.combinations(range(p), s0))
            assert got <= best + 1e-12 * max(1.0, best)


# ------------------------------------------------------------------ init_onb
def test_init_onb_cases():  # test_onb.py:90-126
    np.testing.assert_allclose(S.init_onb(np.eye(4)), np.eye(4), atol=1e-12)
    rng = np.random.default_rng(12)
    q_star = canonical(orth(5, rng))
    np.testing.assert_allclose(S.init_onb(q_star @ np.diag([9.0, 7.0, 5.0, 3.0, 1.0])), q_star,
                               atol=1e-10)
    assert S.orthonormality_defect(S.init_onb(np.random.default_rng(8).standard_normal((8, 64)))) <= 1e-10
    q = S.init_onb(np.random.default_rng(15).standard_normal((8, 3)), rng=np.random.default_rng(0))
    assert q.shape == (8, 8) and S.orthonormality_defect(q) <= 1e-10
    col = np.random.default_rng(16).standard_normal((6, 1))
    assert S.orthonormality_defect(S.init_onb(np.repeat(col, 10, axis=1),
                                              rng=np.random.default_rng(1))) <= 1e-10
    assert S.orthonormality_defect(S.init_onb(np.zeros((5, 7)), rng=np.random.default_rng(2))) <= 1e-10
    ysub = np.random.default_rng(21).standard_normal((7, 2))
    np.testing.assert_array_equal(S.init_onb(ysub, rng=np.random.default_rng(5)),
                                  S.init_onb(ysub, rng=np.random.default_rng(5)))


# ----------------------------------------------------------------- train_onb
def _sparse_signals(rng, q_star, t, s0):
    p = q_star.shape[0]
    x = np.zeros((p, t))
    for j in range(t):
        rows = rng.choice(p, size=s0, replace=False)
        x[rows, j] = rng.uniform(0.5, 2.0, size=s0) * rng.choice([-1, 1], size=s0)
    return q_star @ x


def test_train_onb_contracts():  # test_onb.py:142-214
    rng = np.random.default_rng(30)
    q_star = orth(6, rng)
    y = _sparse_signals(rng, q_star, 64, 2)
    q, code = S.train_onb(y, q_star, 2, 4)
    assert S.frobenius_error(y, q, code) <= 1e-10  # fixed point
    rng = np.random.default_rng(33)
    q0, y = orth(5, rng), rng.standard_normal((5, 20))
    q, code = S.train_onb(y, q0, 2, 0)  # zero rounds: q0 back, its code
    np.testing.assert_array_equal(q, q0)
    ref = S.select_top(q0.T @ y, 2)
    np.testing.assert_array_equal(code.indices, ref.indices)
    np.testing.assert_allclose(code.values, ref.values, rtol=0, atol=1e-14)
    q, code = S.train_onb(np.empty((4, 0)), np.eye(4), 2, 3)  # empty signal set
    np.testing.assert_array_equal(q, np.eye(4))
    assert code.num_columns == 0
    with pytest.raises(ValueError):
        S.train_onb(np.ones((4, 3)), np.eye(5), 2, 1)
    with pytest.raises(ValueError):
        S.train_onb(np.ones((4, 3)), np.eye(4), 2, -1)


def test_train_onb_error_never_increases_and_orthonormal():  # test_onb.py:165, 193; acceptance 02
    rng = np.random.default_rng(44)
    q0, y = orth(8, rng), rng.standard_normal((8, 256))
    errors = []
    for rounds in range(7):
        q, code = S.train_onb(y, q0, 3, rounds)
        errors.append(S.frobenius_error(y, q, code))
        assert S.orthonormality_defect(q) <= 1e-8
    for a, b in zip(errors, errors[1:]):
        assert b <= a + 1e-12 * max(1.0, a)
    q1, c1 = S.train_onb(y, q0, 3, 5)
    q2, c2 = S.train_onb(y.copy(), q0.copy(), 3, 5)  # determinism
    np.testing.assert_array_equal(q1, q2)
    np.testing.assert_array_equal(c1.values, c2.values)


def test_polar_update_never_hurts_fixed_code():  # test_onb.py:178, acceptance 03
    rng = np.random.default_rng(47)
    for _ in range(6):
        q0, y = orth(7, rng), rng.standard_normal((7, 60))
        code = S.select_top(q0.T @ y, 3)
        q1 = S.procrustes_polar(S.sparse_outer(y, code))
        before, after = S.frobenius_error(y, q0, code), S.frobenius_error(y, q1, code)
        assert after <= before + 1e-12 * max(1.0, before)


# -------------------------------------------------------------------- linalg
def test_procrustes_cases():  # test_linalg.py:121-160
    np.testing.assert_allclose(S.procrustes_polar(np.eye(5)), np.eye(5), atol=1e-12)
    np.testing.assert_allclose(S.procrustes_polar(np.diag([3.0, 1.0, 2.0])), np.eye(3), atol=1e-12)
    rng = np.random.default_rng(5)
    u, h = orth(6, rng), orth(6, rng)
    a = u @ (h @ np.diag([5.0, 4.0, 3.0, 2.0, 1.5, 1.0]) @ h.T)
    np.testing.assert_allclose(S.procrustes_polar(a), u, atol=1e-10)
    p = rng.standard_normal((6, 6))
    q = S.procrustes_polar(p)
    assert S.orthonormality_defect(q) <= 1e-10
    best = np.trace(q.T @ p)
    for _ in range(50):
        assert np.trace(orth(6, rng).T @ p) <= best + 1e-10
    low = np.outer(rng.standard_normal(5), rng.standard_normal(5))  # rank one
    assert S.orthonormality_defect(S.procrustes_polar(low)) <= 1e-10
    with pytest.raises(ValueError):
        S.procrustes_polar(np.ones((3, 4)))


def test_thin_svd_cases():  # test_linalg.py:22-95
    r = S.thin_svd(np.eye(3))
    np.testing.assert_allclose(r.sigma, np.ones(3), atol=1e-12)
    r = S.thin_svd(np.array([[3.0, 0.0], [0.0, -2.0]]))
    np.testing.assert_allclose(r.sigma, [3.0, 2.0], atol=1e-12)
    rng = np.random.default_rng(7)
    a = rng.standard_normal((6, 9))
    r = S.thin_svd(a)
    np.testing.assert_allclose((r.u * r.sigma) @ r.v.T, a, atol=1e-9)
    assert S.orthonormality_defect(r.u) <= 1e-10
    assert np.all(np.diff(r.sigma) <= 0)
    eigs = np.sort(np.linalg.eigvalsh(a @ a.T))[::-1]  # test_linalg.py:81 eigen oracle
    np.testing.assert_allclose(r.sigma, np.sqrt(np.maximum(eigs, 0)), atol=1e-10)
    piv = np.argmax(np.abs(r.u), axis=0)  # sign convention: largest |entry| non-negative
    assert np.all(r.u[piv, np.arange(r.u.shape[1])] >= 0)
    r2 = S.thin_svd(a.copy())
    np.testing.assert_array_equal(r.u, r2.u)
    for bad in (np.array([[np.nan, 1.0], [0.0, 1.0]]), np.empty((0, 3)), np.ones(4)):
        with pytest.raises(ValueError):
            S.thin_svd(bad)


# -------------------------------------------------------------- block energy
def test_block_energy_cases():  # test_sbo.py:42-68
    e1 = np.array([1.0, 0.0])
    assert S.block_energy(e1, np.eye(2), 1, "squared-sum") == pytest.approx(1.0)
    assert S.block_energy(e1, np.eye(2), 1, "abs-sum") == pytest.approx(1.0)
    y = np.array([3.0, 4.0])
    assert S.block_energy(y, np.eye(2), 2, "squared-sum") == pytest.approx(25.0)
    assert S.block_energy(y, np.eye(2), 2, "abs-sum") == pytest.approx(7.0)
    rng = np.random.default_rng(3)
    q = orth(6, rng)
    for _ in range(10):
        y = rng.standard_normal(6)
        assert S.block_energy(y, q, 3, "squared-sum") <= np.sum(y ** 2) + 1e-12
    y = q[:, 1] * 2.0 - q[:, 4]
    assert S.block_energy(y, q, 2, "squared-sum") == pytest.approx(float(np.sum(y ** 2)), abs=1e-12)
    with pytest.raises(ValueError):
        S.block_energy(np.ones(2), np.eye(2), 1, "other")


@pytest.mark.parametrize("p,s0", [(64, 8), (64, 3), (256, 16)])
def test_block_energy_tensor_core_shapes_exact(p, s0):
    """p = 64 / 256 (the shapes whose representation runs on the tensor cores):
    block_energy is the exact float64 value (oracle energy_of, sbo.py:126-135)
    for both kinds, not the float32 certificate score."""
    from oracle import sbo_oracle as O
    rng = np.random.default_rng(p + s0)
    q = orth(p, rng)
    for _ in range(4):
        y = rng.standard_normal(p)
        for kind in ("squared-sum", "abs-sum"):
            ref = O.energy_of(y, q, s0, kind)
            assert S.block_energy(y, q, s0, kind) == pytest.approx(ref, rel=1e-12)


# ----------------------------------------------------------------- represent
def test_represent_contracts():  # test_sbo.py:71-165
    rng = np.random.default_rng(70)
    p, m = 8, 300
    one = S.UnionDictionary([orth(p, rng)])
    a, _ = S.represent(rng.standard_normal((p, m)), one, 2)
    assert np.all(a.block == 0)
    d = S.UnionDictionary([orth(p, rng) for _ in range(4)])
    y = d.blocks[2][:, [1, 5]] @ np.array([1.5, -0.7])  # exactly 2-sparse in block 2
    a, code = S.represent(y[:, None], d, 2)
    assert a.block[0] == 2 and a.residual_sq[0] <= 1e-20
    y = rng.standard_normal((p, m))
    a, code = S.represent(y, d, 3)
    for scale in (0.5, 3.0):  # positive scaling keeps the choice
        a2, _ = S.represent(y * scale, d, 3)
        np.testing.assert_array_equal(a.block, a2.block)
    kept = np.sum(code.values ** 2, axis=0)  # residual = ||y||^2 - kept
    np.testing.assert_allclose(a.residual_sq, np.maximum(np.sum(y ** 2, axis=0) - kept, 0.0),
                               rtol=1e-9, atol=1e-12)
    with pytest.raises(ValueError):
        S.represent(np.ones((p + 1, 3)), d, 2)
    bad = y.copy()
    bad[0, 0] = np.nan
    with pytest.raises(ValueError, match="NaN"):
        S.represent(bad, d, 2)


# ------------------------------------------------------- worst set / grouping
def test_worst_set_and_grouping_contracts():  # test_sbo.py:169-250
    def asg(res, blocks=None):
        res = np.asarray(res, np.float64)
        b = np.zeros(res.size, np.int64) if blocks is None else np.asarray(blocks)
        return S.Assignment(b, np.zeros(res.size), res)
    np.testing.assert_array_equal(S.worst_set(asg([0.1, 0.9, 0.3]), 1), [1])
    np.testing.assert_array_equal(S.worst_set(asg([0.5, 0.5, 0.2, 0.5]), 2), [0, 1])
    np.testing.assert_array_equal(np.sort(S.worst_set(asg([0.2, 0.1]), 5)), [0, 1])
    r = np.random.default_rng(2).uniform(size=500)
    np.testing.assert_array_equal(S.worst_set(asg(r), 37), np.argsort(-r, kind="stable")[:37])
    with pytest.raises(ValueError):
        S.worst_set(asg(r), 0)
    y = np.random.default_rng(3).standard_normal((4, 9))
    blocks = np.array([2, 0, 2, 1, 0, 0, 2, 1, 2])
    grouped, ranges, perm = S.group_by_block(y, asg(np.zeros(9), blocks), 4)  # (y, ranges, perm)
    np.testing.assert_array_equal(perm, np.argsort(blocks, kind="stable"))
    np.testing.assert_array_equal(grouped, y[:, perm])
    assert ranges[3] == (9, 9)  # empty block: empty range


# ----------------------------------------------------------------- sbo_train
@pytest.fixture(scope="module")
def scene_signals():
    return data.extract_patches(signals.scene(128, 128, 0),
                                data.PatchConfig(patch_edge=8, count=3000, seed=11))


def test_sbo_train_determinism_monotone_and_report(scene_signals):  # test_sbo.py:297-360; acc 06, 09
    cfg = S.SboConfig(s0=6, k0=2, p0=800, rounds=4, k_max=6, seed=3)
    d1, c1, a1, r1 = S.sbo_train(scene_signals, cfg, workers=1)
    d2, c2, a2, r2 = S.sbo_train(scene_signals, S.SboConfig(**{**cfg.__dict__, "chunk_size": 97}),
                                 workers=7)
    for q1, q2 in zip(d1.blocks, d2.blocks):
        np.testing.assert_array_equal(q1, q2)
    np.testing.assert_array_equal(c1.values, c2.values)
    assert d1.num_blocks == 6 and len(r1.rows) == 6 - 2 + 1  # one block per iteration
    rm = [row.rmse for row in r1.rows]
    assert all(b <= a + 1e-12 for a, b in zip(rm, rm[1:]))
    assert r1.rmse_recomputed == pytest.approx(r1.rmse_final, rel=1e-9)
    for q in d1.blocks:
        assert S.orthonormality_defect(q) <= 1e-8
    _, _, _, rabs = S.sbo_train(scene_signals, S.SboConfig(**{**cfg.__dict__, "energy_kind": "abs-sum",
                                                              "k_max": 3}))
    assert len(rabs.rows) == 2
    with pytest.raises(ValueError):
        S.SboConfig(s0=0).validate()


def test_persistence_round_trip(scene_signals, tmp_path):  # acceptance 11
    cfg = S.SboConfig(s0=6, k0=2, p0=800, rounds=3, k_max=4, seed=5)
    d, code, a, _ = S.sbo_train(scene_signals, cfg)
    store.save_dictionary(tmp_path, d)
    store.save_sbo_codes(tmp_path, code)
    d2, header = store.load_dictionary(tmp_path)
    assert header == {"format": "union-onb", "p": 64, "blocks": 4}
    for q1, q2 in zip(d.blocks, d2.blocks):
        np.testing.assert_array_equal(q1, q2)
    c2 = store.load_sbo_codes(tmp_path)
    for name in ("block", "indices", "values", "energy", "residual_sq"):
        np.testing.assert_array_equal(getattr(code, name), getattr(c2, name))
    a2, k2 = S.represent(scene_signals, d2, 6)  # the reloaded dictionary represents identically
    np.testing.assert_array_equal(a2.block, code.block)
    np.testing.assert_array_equal(k2.indices, code.indices)
