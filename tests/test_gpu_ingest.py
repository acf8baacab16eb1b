"""GPU parity of device-side signal ingestion (data.py:182-208).

Bit-exact against the real reference's extract_patches (golden fixture), against
the benchmark's float32 workload, and through sbo_train: training on device rows
equals training on the same host matrix.
"""
import json

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import sbo_oracle as O

pytestmark = pytest.mark.gpu

import paper_1412_4944_b200 as S  # noqa: E402
from paper_1412_4944_b200 import data, signals  # noqa: E402


def test_extract_patches_matches_reference_bit_for_bit():
    g = golden("ingest_patches")
    for i, (kind, e, norm, count, seed) in enumerate(json.loads(str(g["cases_json"]))):
        cfg = data.PatchConfig(patch_edge=e, count=count, seed=seed, normalization=norm)
        y = data.extract_patches(g[f"grid_{kind}"], cfg)
        assert y.flags.f_contiguous and y.dtype == np.float64 and y.shape == (e * e, count)
        np.testing.assert_array_equal(y, g[f"case{i}"], err_msg=f"case {i}")


@pytest.mark.parametrize("edge,norm", [(8, "unit-range-dc-removed"), (16, "unit-range-dc-removed"),
                                       (7, "unit-range"), (32, "unit-range-dc-removed")])
def test_extract_patches_matches_oracle_large(edge, norm):
    grid = signals.scene(300, 260, 5)
    cfg = data.PatchConfig(patch_edge=edge, count=3000, seed=21, normalization=norm)
    np.testing.assert_array_equal(data.extract_patches(grid, cfg),
                                  O.extract_patches(grid, edge, 3000, 21, norm))


def test_float32_rows_are_the_benchmark_workload():
    grid = signals.scene(512, 512, 0)
    cfg = data.PatchConfig(patch_edge=8, count=8192, seed=11)
    sig = data.extract_patches_device(grid, cfg, dtype=torch.float32)
    want = signals.unit_range(signals.patch_bytes(grid, 8, 8192, 11))
    assert sig.y.dtype == torch.float32
    np.testing.assert_array_equal(sig.y.cpu().numpy(), want)


def test_sbo_train_on_device_rows_equals_host_matrix():
    grid = signals.scene(256, 256, 2)
    pcfg = data.PatchConfig(patch_edge=8, count=4096, seed=3)
    cfg = S.SboConfig(s0=8, k0=3, p0=1024, rounds=3, k_max=5, seed=1)
    host = data.extract_patches(grid, pcfg)
    d1, c1, a1, r1 = S.sbo_train(host, cfg)
    d2, c2, a2, r2 = S.sbo_train(data.extract_patches_device(grid, pcfg), cfg)
    assert d1.num_blocks == d2.num_blocks == 5
    for q1, q2 in zip(d1.blocks, d2.blocks):
        np.testing.assert_array_equal(q1, q2)
    np.testing.assert_array_equal(a1.block, a2.block)
    np.testing.assert_array_equal(c1.indices, c2.indices)
    assert [r.rmse for r in r1.rows] == [r.rmse for r in r2.rows]


def test_represent_accepts_device_rows():
    grid = signals.scene(128, 128, 4)
    pcfg = data.PatchConfig(patch_edge=8, count=2000, seed=8, normalization="unit-range-dc-removed")
    host = data.extract_patches(grid, pcfg)
    rng = np.random.default_rng(0)
    d = S.UnionDictionary([np.linalg.qr(rng.standard_normal((64, 64)))[0] for _ in range(3)])
    a1, c1 = S.represent(host, d, 8)
    a2, c2 = S.represent(data.extract_patches_device(grid, pcfg), d, 8)
    np.testing.assert_array_equal(a1.block, a2.block)
    np.testing.assert_array_equal(c1.values, c2.values)


def test_extract_patches_errors():
    grid = signals.scene(64, 64, 0)
    with pytest.raises(ValueError, match="normalization must be one of"):
        data.extract_patches(grid, data.PatchConfig(normalization="zscore"))
    with pytest.raises(ValueError, match="smaller than a 8x8 patch"):
        data.extract_patches(grid[:5], data.PatchConfig(patch_edge=8, count=4))
    with pytest.raises(ValueError, match="expected a 2-D grayscale grid"):
        data.extract_patches(np.zeros((4, 4, 3), np.uint8), data.PatchConfig(patch_edge=2, count=4))
    with pytest.raises(ValueError, match="count must be at least 1"):
        data.extract_patches(grid, data.PatchConfig(count=0))
    with pytest.raises(ValueError, match="float32 rows"):
        data.extract_patches_device(grid, data.PatchConfig(normalization="unit-range-dc-removed"),
                                    dtype=torch.float32)
