"""The p = 256 tensor-core representation pass (config D shape; tc_energy256.cu):
decisions and kept values equal the oracle's float64 ones on patch data and on
Gaussian data, for both energy kinds, odd block counts (the two epilogue groups
alternate blocks across tiles), partial last tiles and s0 from 4 to 32."""
import numpy as np
import pytest

from oracle import sbo_oracle as O

pytestmark = pytest.mark.gpu

import paper_1412_4944_b200 as S  # noqa: E402
from paper_1412_4944_b200 import data, signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402


def _patches(m, seed):
    grid = signals.scene(256, 256, seed)
    return data.extract_patches(grid, data.PatchConfig(patch_edge=16, count=m, seed=seed + 1))


@pytest.mark.parametrize("kind", ["squared-sum", "abs-sum"])
@pytest.mark.parametrize("K,s0,m,src", [(9, 16, 1000, "patch"), (4, 4, 700, "gauss"),
                                        (3, 32, 300, "patch"), (32, 16, 2000, "gauss")])
def test_tc256_represent_matches_oracle(kind, K, s0, m, src):
    rng = np.random.default_rng(K * 100 + s0)
    qs = [np.linalg.qr(rng.standard_normal((256, 256)))[0] for _ in range(K)]
    y = _patches(m, K) if src == "patch" else rng.standard_normal((256, m))
    eng = Engine(Signals.from_reference(y, require_device()), s0, kind, k_cap=K)
    assert eng.tc, "p = 256 must take the tensor-core pass"
    a, c = S.represent(y, S.UnionDictionary(qs), s0, kind=kind)
    r = O.code_signals(y, qs, s0, kind)
    np.testing.assert_array_equal(a.block, r.block)
    np.testing.assert_array_equal(c.indices, r.indices)
    np.testing.assert_allclose(c.values, r.values, atol=1e-11)
    np.testing.assert_allclose(a.energy, r.energy, rtol=1e-11)
    np.testing.assert_allclose(a.residual_sq, r.residual_sq, rtol=1e-9, atol=1e-12)


def test_tc256_incremental_append_matches_full_pass():
    """represent #1 form: an appended block re-decides only against the stored scores."""
    rng = np.random.default_rng(5)
    K, s0, m = 6, 16, 1500
    qs = [np.linalg.qr(rng.standard_normal((256, 256)))[0] for _ in range(K)]
    y = _patches(m, 3)
    dev = require_device()
    eng = Engine(Signals.from_reference(y, dev), s0, k_cap=K)
    eng.set_blocks(np.stack(qs[:-1]))
    eng.represent_full()
    eng.ensure_capacity(K)
    eng.blocks[K - 1].copy_(__import__("torch").as_tensor(qs[-1]))
    eng.K = K
    eng.energy(K - 1, K, True)
    r = O.code_signals(y, qs, s0)
    np.testing.assert_array_equal(eng.state.best.cpu().numpy(), r.block)
