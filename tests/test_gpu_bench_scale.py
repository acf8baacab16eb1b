"""GPU parity at the benchmarked configurations (BASELINE.json configs B, C, D, E).

The bench's numbers rest on these: each test builds its workload exactly as
bench.py does (seeded procedural scene, 8x8 / 16x16 patches, device sbo_init,
a full representation) and checks one SBO iteration (sbo.py:352-397) against
the CPU oracle.

Contract:
  * worst set: bit-exact as a set (oracle selection on the same residuals);
  * block decisions: bit-exact, except float64 near-ties whose energy gap is
    below 1e-12 relative (counted and bounded here);
  * blocks: max |dQ| <= 1e-9 after the iteration; residuals 1e-9 relative;
    RMSE 1e-10 relative against the oracle's recomputation.
Config C (m = 2^24) is checked on seeded random 2^17-signal subsets for the
per-signal stages (each signal is independent there) and in full for the worst
set, the new block and one retrained block.
"""
import os

import numpy as np
import pytest
import torch

from oracle import sbo_oracle as O

pytestmark = pytest.mark.gpu

from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _block_rng, _init_into  # noqa: E402

WORKERS = os.cpu_count() or 1
NEAR_TIE = 1e-12


@pytest.fixture(scope="module")
def dev():
    return require_device()


def check_decisions(y64, blocks, s0, got, want, tol=NEAR_TIE, max_frac=1e-4, kind="squared-sum"):
    """got == want except where the two chosen blocks' float64 energies (oracle
    arithmetic) are within tol relative: those are the documented near-ties."""
    bad = np.flatnonzero(np.asarray(got) != np.asarray(want))
    for j in bad:
        e_got = O.energy_of(y64[:, j], blocks[got[j]], s0, kind)
        e_want = O.energy_of(y64[:, j], blocks[want[j]], s0, kind)
        assert abs(e_got - e_want) <= tol * max(abs(e_want), 1e-300), \
            (int(j), int(got[j]), int(want[j]), e_got, e_want)
    assert bad.size <= max(1, int(max_frac * len(got))), bad.size
    return bad.size


def bench_workload(dev, m, scene, edge, K, s0, rounds=6, lo=0, hi=None):
    """The bench's entering state: rows, engine after device sbo_init(k0 = K-1) and
    a full representation, and the new block's draws."""
    grid = signals.scene(scene, scene, 0)
    rows = signals.unit_range(signals.patch_bytes(grid, edge, m, 11, lo, hi))
    eng = Engine(Signals.from_rows(rows, dev), s0, k_cap=K)
    cfg = SboConfig(s0=s0, k0=K - 1, p0=4096, rounds=rounds, k_max=K, seed=1)
    _init_into(eng, cfg, m)
    eng.represent_full()
    draws = _block_rng(1, 1, K - 1).standard_normal((edge * edge + 8, edge * edge))
    return rows, eng, draws


class Rep1Hook:
    """Records the assignment and blocks at the first grouping of an iteration
    (i.e. right after represent #1, sbo.py:361-367)."""

    def __init__(self, eng):
        self.eng, self.best, self.blocks = eng, None, None
        self.orig = eng.group

    def __call__(self, K):
        if self.best is None:
            self.best = self.eng.state.best.clone()
            self.blocks = self.eng.blocks[:K].clone()
        return self.orig(K)


def full_iteration_check(dev, rows, eng, draws, s0, rounds, iter_tol=1e-9):
    """One iteration on the GPU and in the oracle from the same entering state."""
    K0 = eng.K
    m, p = rows.shape
    y64 = rows.T.astype(np.float64)
    entering = [q for q in eng.blocks[:K0].cpu().numpy()]
    res_in = eng.state.residual.cpu().numpy()
    rep0 = O.code_signals(y64, entering, s0, workers=WORKERS)
    n0 = check_decisions(y64, entering, s0, eng.state.best.cpu().numpy(), rep0.block)
    np.testing.assert_allclose(res_in, rep0.residual_sq, rtol=1e-9, atol=1e-12)
    w = max(p, m // 16)
    hook = Rep1Hook(eng)
    eng.group = hook
    out = eng.iterate(w, rounds, draws)
    eng.group = hook.orig
    # the oracle from the GPU's entering residuals (teacher-forced entering state)
    tr = O.iterate(y64, entering, res_in, s0, rounds, w, seed=1, workers=WORKERS)
    np.testing.assert_array_equal(np.sort(out.worst.cpu().numpy()), np.sort(tr.worst))
    # represent #1 against the oracle on the GPU's new block (exact decisions)
    blocks1 = [q for q in hook.blocks.cpu().numpy()]
    rep1 = O.code_signals(y64, blocks1, s0, workers=WORKERS)
    n1 = check_decisions(y64, blocks1, s0, hook.best.cpu().numpy(), rep1.block)
    assert np.abs(blocks1[K0] - tr.new_block).max() <= iter_tol
    got = [q for q in eng.blocks[: eng.K].cpu().numpy()]
    dq = max(np.abs(a - b).max() for a, b in zip(got, tr.blocks))
    assert dq <= iter_tol, dq
    # represent #2 against the oracle on the GPU's final blocks (exact decisions)
    rep2 = O.code_signals(y64, got, s0, workers=WORKERS)
    best = eng.state.best.cpu().numpy()
    n2 = check_decisions(y64, got, s0, best, rep2.block)
    np.testing.assert_allclose(eng.state.residual.cpu().numpy(), rep2.residual_sq,
                               rtol=1e-9, atol=1e-12)
    assert out.rmse == pytest.approx(O.rmse_of(rep2.residual_sq, p, m), rel=1e-10)
    # and against the oracle's own trajectory (its blocks differ by <= dq)
    assert out.rmse == pytest.approx(tr.rmse, rel=1e-8)
    return {"dq": dq, "near_ties": (n0, n1, n2), "rmse": out.rmse}


def test_config_b_full_iteration(dev):
    """Config B exactly as bench.py --m 2^20 builds it: 2048^2 scene, m = 2^20,
    device sbo_init (k0 = 15), 15 -> 16 blocks, s0 = 8, R = 6, W = m/16."""
    rows, eng, draws = bench_workload(dev, 1 << 20, 2048, 8, 16, 8)
    r = full_iteration_check(dev, rows, eng, draws, 8, 6)
    print("config B:", r)


def test_config_e_k64_full_iteration(dev):
    """Config E's K = 64 branch (more than 32 blocks: no candidate masks in the
    float64 re-decision) through one full iteration, 63 -> 64 blocks."""
    rows, eng, draws = bench_workload(dev, 1 << 17, 1024, 8, 64, 8, rounds=3)
    r = full_iteration_check(dev, rows, eng, draws, 8, 3)
    print("config E K=64:", r)


@pytest.mark.parametrize("s0", [4, 32])
def test_config_e_s0_full_iteration(dev, s0):
    """Config E's s0 extremes (selection networks for s0 = 4, bisection for 32)."""
    rows, eng, draws = bench_workload(dev, 1 << 17, 1024, 8, 16, s0, rounds=3)
    r = full_iteration_check(dev, rows, eng, draws, s0, 3)
    print(f"config E s0={s0}:", r)


def test_config_d_full_iteration(dev):
    """Config D's shape: p = 256 (16x16 patches), 31 -> 32 blocks, s0 = 16, at
    m = 2^18 (the p = 256 tensor-core energy pass, its certificate and the
    float64 re-decision, the general-p rounds and the 256x256 polar)."""
    rows, eng, draws = bench_workload(dev, 1 << 18, 2048, 16, 32, 16, rounds=2)
    r = full_iteration_check(dev, rows, eng, draws, 16, 2)
    print("config D:", r)


def test_config_c_sampled(dev):
    """Config C at its stated size (m = 2^24, 4096^2 scene) on one GPU:
      * entering and final representations on a seeded 2^17-signal subset;
      * the worst set in full (oracle selection over all 2^24 GPU residuals);
      * the new block (init + 6 rounds on the W = 2^20 worst signals) in full;
      * represent #1 on the subset, and one retrained block on its full group."""
    m, s0, R = 1 << 24, 8, 6
    rows, eng, draws = bench_workload(dev, m, 4096, 8, 16, s0)
    K0, p = eng.K, 64
    entering = [q for q in eng.blocks[:K0].cpu().numpy()]
    sub = np.sort(np.random.default_rng(7).choice(m, 1 << 17, replace=False))
    ysub = rows[sub].T.astype(np.float64)
    res_in = eng.state.residual.cpu().numpy()
    rep0 = O.code_signals(ysub, entering, s0, workers=WORKERS)
    check_decisions(ysub, entering, s0, eng.state.best.cpu().numpy()[sub], rep0.block)
    np.testing.assert_allclose(res_in[sub], rep0.residual_sq, rtol=1e-9, atol=1e-12)
    w = m // 16
    want_worst = O.worst_members(res_in, w)
    hook = Rep1Hook(eng)
    eng.group = hook
    out = eng.iterate(w, R, draws)
    eng.group = hook.orig
    np.testing.assert_array_equal(np.sort(out.worst.cpu().numpy()), np.sort(want_worst))
    # the new block, trained on the worst set from the same seeded draws
    yw = rows[np.sort(want_worst)].T.astype(np.float64)
    q_new, _, _ = O.train_block(yw, O.init_block(yw, O.stream(1, 1, K0)), s0, R)
    dq_new = np.abs(hook.blocks[K0].cpu().numpy() - q_new).max()
    assert dq_new <= 1e-9, dq_new
    del yw
    # represent #1 (incremental: only the new block can win) on the subset
    blocks1 = [q for q in hook.blocks.cpu().numpy()]
    rep1 = O.code_signals(ysub, blocks1, s0, workers=WORKERS)
    best1 = hook.best.cpu().numpy()
    check_decisions(ysub, blocks1, s0, best1[sub], rep1.block)
    # one retrained block on its full group (the median-size nonempty group)
    counts = np.bincount(best1, minlength=K0 + 1)
    nonempty = np.flatnonzero(counts)
    b = int(nonempty[np.argsort(counts[nonempty])[len(nonempty) // 2]])
    yb = rows[np.flatnonzero(best1 == b)].T.astype(np.float64)
    q_b, _, _ = O.train_block(yb, blocks1[b], s0, R)
    dq_b = np.abs(eng.blocks[b].cpu().numpy() - q_b).max()
    assert dq_b <= 1e-9, (b, counts[b], dq_b)
    del yb
    # represent #2 on the subset with the GPU's final blocks
    got = [q for q in eng.blocks[: eng.K].cpu().numpy()]
    rep2 = O.code_signals(ysub, got, s0, workers=WORKERS)
    check_decisions(ysub, got, s0, eng.state.best.cpu().numpy()[sub], rep2.block)
    res2 = eng.state.residual.cpu().numpy()
    np.testing.assert_allclose(res2[sub], rep2.residual_sq, rtol=1e-9, atol=1e-12)
    # the RMSE is the deterministic sum of the per-signal residuals
    assert out.rmse == pytest.approx(float(np.sqrt(res2.sum() / (p * m))), rel=1e-12)
    print(f"config C: dq_new={dq_new:.2e} block {b} ({counts[b]} signals) dq={dq_b:.2e} "
          f"rmse={out.rmse:.6e}")


# ------------------------------------------------------- adversarial certificate
def _rotation(p, theta, rng):
    """A rotation by theta in a random plane."""
    u, v = np.linalg.qr(rng.standard_normal((p, 2)))[0].T
    r = np.eye(p)
    for a, b in ((u, v),):
        r += (np.cos(theta) - 1) * (np.outer(a, a) + np.outer(b, b)) + \
            np.sin(theta) * (np.outer(b, a) - np.outer(a, b))
    return r


@pytest.mark.parametrize("p,s0", [(64, 8), (256, 16)])
def test_certificate_near_tied_blocks(dev, p, s0):
    """Blocks whose energies are within ~1e-7 of each other for every signal
    (a block and a slightly rotated copy), an exact duplicate (ties -> lowest
    index), and signals with many equal-magnitude coefficients (cancellation at
    the selection boundary): the tensor-core pass must flag these and the
    float64 re-decision must reproduce the oracle's decisions."""
    rng = np.random.default_rng(11 + p)
    m = 8192
    q0 = np.linalg.qr(rng.standard_normal((p, p)))[0]
    q1 = q0 @ _rotation(p, 1e-7, rng)
    q1 = np.linalg.qr(q1)[0] * np.sign(np.diag(np.linalg.qr(q1)[1]))
    q3 = np.linalg.qr(rng.standard_normal((p, p)))[0]
    blocks = [q0, q1, q0.copy(), q3]
    v = rng.standard_normal((p, m))
    # a third of the signals: s0 + 1 equal-magnitude coefficients (ties at the
    # selection boundary) plus a 1e-9 perturbation on some of them
    tie = rng.random(m) < 1 / 3
    for j in np.flatnonzero(tie):
        c = np.zeros(p)
        at = rng.choice(p, s0 + 1, replace=False)
        c[at] = rng.choice([-1.0, 1.0], s0 + 1)
        if rng.random() < 0.5:
            c += 1e-9 * rng.standard_normal(p)
        v[:, j] = c
    y = np.where(tie[None, :], q0 @ v, v)
    y32 = np.ascontiguousarray(y.T.astype(np.float32))
    y64 = y32.T.astype(np.float64)
    eng = Engine(Signals.from_rows(y32, dev), s0, k_cap=len(blocks))
    eng.set_blocks(np.stack(blocks))
    eng.represent_full()
    rep = O.code_signals(y64, blocks, s0, workers=WORKERS)
    n = check_decisions(y64, blocks, s0, eng.state.best.cpu().numpy(), rep.block)
    np.testing.assert_allclose(eng.state.residual.cpu().numpy(), rep.residual_sq, rtol=1e-9,
                               atol=1e-12)
    # the duplicate (block 2) never wins over block 0
    assert not (eng.state.best.cpu().numpy() == 2).any()
    print(f"p={p}: {n} float64 near-ties, flagged {int(eng.nflag.item())}")


@pytest.mark.parametrize("p,s0", [(64, 8), (256, 16)])
@pytest.mark.parametrize("perturb", [0.0, 1e-9])
def test_incremental_append_of_near_copy(dev, p, s0, perturb):
    """represent #1 (accumulate mode): the appended block is a copy (or a 1e-9
    rotation) of an existing block.  A flagged signal must keep its incoming exact
    winner for the float64 re-decision, so the first maximum wins (sbo.py:191)."""
    rng = np.random.default_rng(5 + p)
    m = 16384
    blocks = [np.linalg.qr(rng.standard_normal((p, p)))[0] for _ in range(3)]
    y32 = rng.standard_normal((m, p)).astype(np.float32)
    y64 = y32.T.astype(np.float64)
    eng = Engine(Signals.from_rows(y32, dev), s0, k_cap=4)
    eng.set_blocks(np.stack(blocks))
    eng.represent_full()
    new = blocks[1] if perturb == 0.0 else blocks[1] @ _rotation(p, perturb, rng)
    eng.blocks[3].copy_(torch.from_numpy(np.ascontiguousarray(new)))
    eng.K = 4
    eng.energy(3, 4, True)
    allb = blocks + [new]
    rep = O.code_signals(y64, allb, s0, workers=WORKERS)
    got = eng.state.best.cpu().numpy()
    check_decisions(y64, allb, s0, got, rep.block)
    if perturb == 0.0:
        assert not (got == 3).any()  # an exact copy never wins (ties -> lower block)
