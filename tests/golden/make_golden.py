"""Generate the golden fixtures from the REAL reference (``orthodict``).

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src, runs it on
seeded inputs and writes small ``.npz`` fixtures next to this script.  The
fixtures pin the CPU oracle (tests/test_oracle_golden.py) and are the parity
targets of the GPU tests.  Signals are float32-rounded before the reference sees
them (upcast to float64), exactly what the device holds.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import orthodict  # noqa: E402
from orthodict import data as rdata  # noqa: E402
from orthodict import linalg as rlinalg  # noqa: E402
from orthodict import onb as ronb  # noqa: E402
from orthodict import sbo as rsbo  # noqa: E402

from paper_1412_4944_b200 import signals  # noqa: E402


def _f32(y):
    return np.asarray(y, np.float32).astype(np.float64)


def _orth(p, rng):
    q, _ = np.linalg.qr(rng.standard_normal((p, p)))
    return q


def desk_signals():
    """conftest.py:6-26 desk fixture: 512x512 scene seed 0, 8x8 patches, m=8192, seed 11."""
    grid = rdata.synthetic_test_image(512, 512, seed=0)
    y = rdata.extract_patches(grid, rdata.PatchConfig(patch_edge=8, count=8192, seed=11))
    u8 = np.rint(y.T * 255.0).astype(np.uint8)  # (m, p) rows
    assert np.array_equal(u8.astype(np.float64).T / 255.0, y)
    return grid, u8


def make_patches():
    grid, u8 = desk_signals()
    np.savez_compressed(HERE / "desk_patches.npz", u8=u8,
                        grid_sum=np.int64(grid.astype(np.int64).sum()),
                        grid_head=grid[:4, :16])
    return u8


def make_represent(u8):
    y = _f32(u8.T / 255.0)  # p x m float64 of the float32 signals
    cfg = rsbo.SboConfig(s0=8, k0=4, p0=4096, rounds=6, seed=1)
    d = rsbo.sbo_init(y, cfg, workers=1)
    out = {"blocks": np.stack(d.blocks)}
    for kind in ("squared-sum", "abs-sum"):
        a, code = rsbo.represent(y, d, 8, kind=kind, workers=1)
        tag = "sq" if kind == "squared-sum" else "abs"
        out[f"{tag}_block"] = a.block.astype(np.int16)
        out[f"{tag}_energy"] = a.energy
        out[f"{tag}_residual"] = a.residual_sq
        out[f"{tag}_indices"] = code.indices.astype(np.uint8)
        out[f"{tag}_values"] = code.values
    np.savez_compressed(HERE / "desk_represent.npz", **out)
    return d, y


def make_iteration(d, y):
    """One teacher-forced iteration (sbo.py:352-397) entering with 4 blocks."""
    p, m = y.shape
    a, _ = rsbo.represent(y, d, 8, workers=1)
    w = max(p, m // 16)
    blocks = [q.copy() for q in d.blocks]
    worst = rsbo.worst_set(a, w)
    rng = rsbo._block_rng(1, 1, len(blocks))
    ysub = y[:, worst]
    q0 = ronb.init_onb(ysub, rng=rng)
    hist = []
    q = q0
    for r in range(6):
        q, _ = ronb.train_onb(ysub, q, 8, 1)
        hist.append(q)
    blocks.append(q)
    a1, c1 = rsbo.represent(y, rsbo.UnionDictionary(blocks), 8, workers=1)
    grouped, ranges, perm = rsbo.group_by_block(y, a1, len(blocks))
    retrained = []
    for b, (s, e) in enumerate(ranges):
        retrained.append(blocks[b] if s == e else ronb.train_onb(grouped[:, s:e], blocks[b], 8, 6)[0])
    a2, c2 = rsbo.represent(y, rsbo.UnionDictionary(retrained), 8, workers=1)
    np.savez_compressed(
        HERE / "desk_iteration.npz",
        entering=np.stack(d.blocks), entering_residual=a.residual_sq,
        worst=worst.astype(np.int32), init_block=q0, new_block_rounds=np.stack(hist),
        rep1_block=a1.block.astype(np.int16), rep1_indices=c1.indices.astype(np.uint8),
        rep1_values=c1.values,
        ranges=np.array(ranges, np.int64), retrained=np.stack(retrained),
        rep2_block=a2.block.astype(np.int16), rep2_residual=a2.residual_sq,
        rep2_energy=a2.energy,
        rmse=np.float64(np.sqrt(a2.residual_sq.sum() / (p * m))))


def make_gaussian_iteration():
    """Gaussian near-tie stress: p=64, entering K-1=15 random blocks, m=16384."""
    p, m, k = 64, 16384, 16
    y = _f32(signals.gaussian_signals(p, m, seed=5).T)
    rng = np.random.default_rng(123)
    blocks = [_orth(p, rng) for _ in range(k - 1)]
    d = rsbo.UnionDictionary(blocks)
    a, c = rsbo.represent(y, d, 8, workers=1)
    w = max(p, m // 16)
    worst = rsbo.worst_set(a, w)
    rr = rsbo._block_rng(0, 1, len(blocks))
    ysub = y[:, worst]
    qn, _ = ronb.train_onb(ysub, ronb.init_onb(ysub, rng=rr), 8, 6)
    nb = blocks + [qn]
    a1, _ = rsbo.represent(y, rsbo.UnionDictionary(nb), 8, workers=1)
    grouped, ranges, _ = rsbo.group_by_block(y, a1, len(nb))
    rt = [nb[b] if s == e else ronb.train_onb(grouped[:, s:e], nb[b], 8, 6)[0]
          for b, (s, e) in enumerate(ranges)]
    a2, _ = rsbo.represent(y, rsbo.UnionDictionary(rt), 8, workers=1)
    np.savez_compressed(
        HERE / "gauss_iteration.npz", entering=np.stack(blocks),
        rep0_block=a.block.astype(np.int16), rep0_residual=a.residual_sq,
        rep0_indices=c.indices.astype(np.uint8), rep0_values=c.values,
        worst=worst.astype(np.int32), new_block=qn, rep1_block=a1.block.astype(np.int16),
        retrained=np.stack(rt), rep2_block=a2.block.astype(np.int16),
        rep2_residual=a2.residual_sq)


def make_train(u8):
    """Config A: sbo_train(k0=4, k_max=14) on the desk fixture, 10 iterations."""
    y = _f32(u8.T / 255.0)
    cfg = rsbo.SboConfig(s0=8, k0=4, p0=4096, rounds=6, k_max=14, seed=0)
    d, code, a, rep = rsbo.sbo_train(y, cfg, workers=1)
    np.savez_compressed(
        HERE / "desk_train.npz", rmse=np.array([r.rmse for r in rep.rows]),
        sizes=np.array([r.dictionary_size for r in rep.rows]), blocks=np.stack(d.blocks),
        block=code.block.astype(np.int16), rmse_final=np.float64(rep.rmse_final),
        rmse_recomputed=np.float64(rep.rmse_recomputed),
        init_blocks=np.stack(rsbo.sbo_init(y, cfg, workers=1).blocks))


def make_small():
    """Small seeded cases mirroring the reference unit tests (p = 4..8)."""
    out = {}
    rng = np.random.default_rng(7)
    # represent, p=4 K=3 m=100, both kinds (test_sbo.py:87-96)
    qs = np.stack([_orth(4, rng) for _ in range(3)])
    y = rng.standard_normal((4, 100))
    out["rep_blocks"], out["rep_y"] = qs, y
    for kind, tag in (("squared-sum", "sq"), ("abs-sum", "abs")):
        a, c = rsbo.represent(y, rsbo.UnionDictionary(list(qs)), 2, kind=kind, workers=1)
        out[f"rep_{tag}_block"], out[f"rep_{tag}_energy"] = a.block, a.energy
        out[f"rep_{tag}_residual"] = a.residual_sq
        out[f"rep_{tag}_indices"], out[f"rep_{tag}_values"] = c.indices, c.values
    # train_onb p=8 t=256 s0=3 R=6 (acceptance 2)
    q0 = _orth(8, rng)
    yt = rng.standard_normal((8, 256))
    q, c = ronb.train_onb(yt, q0, 3, 6)
    out.update(tr_q0=q0, tr_y=yt, tr_q=q, tr_indices=c.indices, tr_values=c.values)
    # init_onb: wide, too-few-columns (completion), rank one, all zero
    yw = rng.standard_normal((8, 64))
    out.update(init_wide_y=yw, init_wide_q=ronb.init_onb(yw))
    yf = rng.standard_normal((8, 3))
    out.update(init_few_y=yf, init_few_q=ronb.init_onb(yf, rng=np.random.default_rng(0)))
    y1 = np.repeat(rng.standard_normal((6, 1)), 10, axis=1)
    out.update(init_rank1_y=y1, init_rank1_q=ronb.init_onb(y1, rng=np.random.default_rng(1)))
    out.update(init_zero_q=ronb.init_onb(np.zeros((5, 7)), rng=np.random.default_rng(2)))
    # procrustes on seeded 8x8 and a 64x64 well-conditioned P
    pm = rng.standard_normal((8, 8))
    out.update(polar_p8=pm, polar_q8=rlinalg.procrustes_polar(pm))
    p64 = rng.standard_normal((64, 64)) + 4 * np.eye(64)
    out.update(polar_p64=p64, polar_q64=rlinalg.procrustes_polar(p64))
    res = rlinalg.thin_svd(p64)
    out.update(svd64_u=res.u, svd64_s=res.sigma, svd64_v=res.v)
    # worst_set sort oracle (test_sbo.py:182-188)
    r = rng.random(1000)
    out.update(worst_res=r, worst_100=rsbo.worst_set(rsbo.Assignment(
        np.zeros(1000, np.int64), np.zeros(1000), r), 100))
    np.savez_compressed(HERE / "small_cases.npz", **out)


INGEST_CASES = [  # (grid, edge, normalization, count, seed)
    ("u8", 1, "unit-range", 40, 5), ("u8", 3, "unit-range-dc-removed", 50, 6),
    ("u8", 8, "unit-range", 50, 7), ("u8", 8, "unit-range-dc-removed", 50, 8),
    ("u8", 12, "unit-range-dc-removed", 30, 9), ("u8", 16, "unit-range", 30, 10),
    ("u8", 16, "unit-range-dc-removed", 30, 11), ("f64", 5, "unit-range", 40, 12),
    ("f64", 8, "unit-range-dc-removed", 40, 13),
]


def make_ingest():
    """data.py:182-208 extract_patches on a small scene and a float grid (device ingestion)."""
    grids = {"u8": rdata.synthetic_test_image(96, 80, seed=3),
             "f64": np.random.default_rng(4).uniform(0.0, 255.0, (37, 29))}
    import json
    out = {"grid_u8": grids["u8"], "grid_f64": grids["f64"],
           "cases_json": np.array(json.dumps(INGEST_CASES))}
    for i, (g, e, norm, count, seed) in enumerate(INGEST_CASES):
        cfg = rdata.PatchConfig(patch_edge=e, count=count, seed=seed, normalization=norm)
        out[f"case{i}"] = rdata.extract_patches(grids[g], cfg)
    np.savez_compressed(HERE / "ingest_patches.npz", **out)


def make_store():
    """store.py:53-133 files (dictionary union + dense, SBO codes), as bytes."""
    import tempfile
    from orthodict import store as rstore
    rng = np.random.default_rng(17)
    m, k = 37, 5
    code = rsbo.SparseCode(block=rng.integers(0, 3, m), indices=np.sort(rng.integers(0, 16, (k, m)), axis=0),
                           values=rng.standard_normal((k, m)), energy=rng.uniform(0, 2, m),
                           residual_sq=rng.uniform(0, 1, m))
    union = rsbo.UnionDictionary([_orth(4, rng) for _ in range(3)])
    dense = rng.standard_normal((6, 9))
    out = {"block": code.block, "indices": code.indices, "values": code.values,
           "energy": code.energy, "residual_sq": code.residual_sq,
           "union": np.stack(union.blocks), "dense": dense}
    with tempfile.TemporaryDirectory() as t:
        rstore.save_sbo_codes(t, code)
        out["codes_odm"] = np.frombuffer((Path(t) / "codes.odm").read_bytes(), np.uint8)
        out["codes_meta"] = np.array((Path(t) / "codes.meta.json").read_text())
    with tempfile.TemporaryDirectory() as t:
        rstore.save_dictionary(t, union, {"note": "x"})
        out["union_odm"] = np.frombuffer((Path(t) / "dict.odm").read_bytes(), np.uint8)
        out["union_meta"] = np.array((Path(t) / "dict.meta.json").read_text())
    with tempfile.TemporaryDirectory() as t:
        rstore.save_dictionary(t, dense)
        out["dense_odm"] = np.frombuffer((Path(t) / "dict.odm").read_bytes(), np.uint8)
        out["dense_meta"] = np.array((Path(t) / "dict.meta.json").read_text())
    np.savez_compressed(HERE / "store_files.npz", **out)


def main():
    if sys.argv[1:] == ["ingest"]:
        make_ingest()
        return
    if sys.argv[1:] == ["store"]:
        make_store()
        return
    u8 = make_patches()
    d, y = make_represent(u8)
    make_iteration(d, y)
    make_gaussian_iteration()
    make_train(u8)
    make_small()
    make_ingest()
    make_store()
    (HERE / "VERSIONS.txt").write_text(
        f"orthodict {orthodict.__version__}\nnumpy {np.__version__}\n"
        f"scipy {__import__('scipy').__version__}\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
