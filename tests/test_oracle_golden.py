"""Pin the CPU oracle against fixtures produced by the real reference (CPU only)."""
import json

import numpy as np
import pytest

from conftest import golden
from oracle import sbo_oracle as O
from paper_1412_4944_b200 import signals


def test_signal_generator_matches_reference_bytes():
    g = golden("desk_patches")
    grid = signals.scene(512, 512, 0)
    assert int(grid.astype(np.int64).sum()) == int(g["grid_sum"])
    np.testing.assert_array_equal(grid[:4, :16], g["grid_head"])
    np.testing.assert_array_equal(signals.patch_bytes(grid, 8, 8192, 11), g["u8"])


@pytest.mark.parametrize("kind,tag", [("squared-sum", "sq"), ("abs-sum", "abs")])
def test_represent_desk(desk_y64, kind, tag):
    g = golden("desk_represent")
    c = O.code_signals(desk_y64, list(g["blocks"]), 8, kind)
    np.testing.assert_array_equal(c.block, g[f"{tag}_block"])
    np.testing.assert_array_equal(c.indices, g[f"{tag}_indices"])
    np.testing.assert_allclose(c.values, g[f"{tag}_values"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(c.energy, g[f"{tag}_energy"], rtol=1e-12)
    np.testing.assert_allclose(c.residual_sq, g[f"{tag}_residual"], rtol=1e-9, atol=1e-14)


def test_init_blocks_desk(desk_y64):
    g = golden("desk_represent")
    blocks = O.initial_blocks(desk_y64, 8, 4, 4096, 6, seed=1)
    for q, r in zip(blocks, g["blocks"]):
        np.testing.assert_allclose(q, r, atol=1e-12)


def test_iteration_desk(desk_y64):
    g = golden("desk_iteration")
    tr = O.iterate(desk_y64, list(g["entering"]), g["entering_residual"], 8, 6,
                   max(64, 8192 // 16), seed=1)
    np.testing.assert_array_equal(tr.worst, g["worst"])
    np.testing.assert_allclose(tr.new_block, g["new_block_rounds"][-1], atol=1e-11)
    np.testing.assert_array_equal(tr.rep1.block, g["rep1_block"])
    np.testing.assert_array_equal(np.array(tr.ranges), g["ranges"])
    for q, r in zip(tr.blocks, g["retrained"]):
        np.testing.assert_allclose(q, r, atol=1e-11)
    np.testing.assert_array_equal(tr.rep2.block, g["rep2_block"])
    np.testing.assert_allclose(tr.rep2.residual_sq, g["rep2_residual"], rtol=1e-8, atol=1e-13)
    assert tr.rmse == pytest.approx(float(g["rmse"]), rel=1e-12)


def test_iteration_gaussian():
    g = golden("gauss_iteration")
    y = signals.gaussian_signals(64, 16384, seed=5).T.astype(np.float64)
    rep0 = O.code_signals(y, list(g["entering"]), 8)
    np.testing.assert_array_equal(rep0.block, g["rep0_block"])
    np.testing.assert_array_equal(rep0.indices, g["rep0_indices"])
    tr = O.iterate(y, list(g["entering"]), rep0.residual_sq, 8, 6, 1024, seed=0)
    np.testing.assert_array_equal(tr.worst, g["worst"])
    np.testing.assert_allclose(tr.new_block, g["new_block"], atol=1e-11)
    np.testing.assert_array_equal(tr.rep1.block, g["rep1_block"])
    for q, r in zip(tr.blocks, g["retrained"]):
        np.testing.assert_allclose(q, r, atol=1e-11)
    np.testing.assert_array_equal(tr.rep2.block, g["rep2_block"])


def test_train_desk_config_a(desk_y64):
    g = golden("desk_train")
    blocks, rep, rmses, notes = O.train(desk_y64, 8, k0=4, p0=4096, rounds=6, k_max=14, seed=0)
    np.testing.assert_allclose(rmses, g["rmse"], rtol=1e-12)
    assert len(blocks) == 14
    np.testing.assert_array_equal(rep.block, g["block"])


def test_small_cases():
    g = golden("small_cases")
    for kind, tag in (("squared-sum", "sq"), ("abs-sum", "abs")):
        c = O.code_signals(g["rep_y"], list(g["rep_blocks"]), 2, kind)
        np.testing.assert_array_equal(c.block, g[f"rep_{tag}_block"])
        np.testing.assert_array_equal(c.indices, g[f"rep_{tag}_indices"])
        np.testing.assert_allclose(c.energy, g[f"rep_{tag}_energy"], rtol=1e-12)
    q, i, v = O.train_block(g["tr_y"], g["tr_q0"], 3, 6)
    np.testing.assert_allclose(q, g["tr_q"], atol=1e-12)
    np.testing.assert_array_equal(i, g["tr_indices"])
    np.testing.assert_allclose(O.init_block(g["init_wide_y"]), g["init_wide_q"], atol=1e-12)
    np.testing.assert_allclose(O.init_block(g["init_few_y"], np.random.default_rng(0)),
                               g["init_few_q"], atol=1e-12)
    np.testing.assert_allclose(O.init_block(g["init_rank1_y"], np.random.default_rng(1)),
                               g["init_rank1_q"], atol=1e-12)
    np.testing.assert_allclose(O.init_block(np.zeros((5, 7)), np.random.default_rng(2)),
                               g["init_zero_q"], atol=1e-12)
    np.testing.assert_allclose(O.polar(g["polar_p8"]), g["polar_q8"], atol=1e-12)
    np.testing.assert_allclose(O.polar(g["polar_p64"]), g["polar_q64"], atol=1e-12)
    np.testing.assert_array_equal(O.worst_members(g["worst_res"], 100), g["worst_100"])


def test_select_hand_cases():
    i, v = O.top_support(np.array([3.0, -5.0, 1.0, 0.0]), 2)
    assert list(i[:, 0]) == [0, 1] and list(v[:, 0]) == [3.0, -5.0]
    i, v = O.top_support(np.array([1.0, -1.0, 1.0]), 2)
    assert list(i[:, 0]) == [0, 1]
    i, v = O.top_support(np.array([2.0, 0.0, -1.0]), 4)
    assert list(i[:, 0]) == [0, 1, 2]


def test_extract_patches_oracle_matches_reference():
    """The ingestion restatement reproduces data.py:182-208 bit for bit."""
    g = golden("ingest_patches")
    for i, (kind, e, norm, count, seed) in enumerate(json.loads(str(g["cases_json"]))):
        y = O.extract_patches(g[f"grid_{kind}"], e, count, seed, norm)
        np.testing.assert_array_equal(y, g[f"case{i}"], err_msg=f"case {i}")
