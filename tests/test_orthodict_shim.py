"""The reference-side binding (integration/orthodict_b200.py).

Drives the reference's own CLI (``orthodict.cli.main``, cli.py:349-365) through
the shim: exit codes, files written by the reference's own ``store`` from our
results (store.py:53-133 ``isinstance`` checks), and the exception mapping
(cli.py:29-30, 356-364).  ``orthodict`` is imported from ``baseline/_ref`` (the
reference installed offline, which travels to the GPU box) or, in the build
container, from /root/reference/pkg/src; the tests skip when neither exists.
The product package itself never imports ``orthodict`` (tests/test_capi.py).
"""
import importlib
import os
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import REPO, has_cuda

for _cand in (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (_cand / "orthodict").is_dir() and str(_cand) not in sys.path:
        sys.path.append(str(_cand))
        break

orthodict = pytest.importorskip("orthodict")
import orthodict.cli  # noqa: E402
import orthodict.data  # noqa: E402
import orthodict.store  # noqa: E402

sys.path.insert(0, str(REPO / "integration"))
shim = importlib.import_module("orthodict_b200")


@pytest.fixture
def installed():
    shim.install()
    yield shim
    shim.uninstall()


# ------------------------------------------------------------ host logic (CPU)
def test_install_rebinds_every_import_time_binding(installed):
    import orthodict.linalg
    import orthodict.sbo
    assert orthodict.cli.sbo_train is shim.sbo_train
    assert orthodict.cli.represent is shim.represent
    assert orthodict.cli.frobenius_error is shim.frobenius_error
    assert orthodict.sbo_train is shim.sbo_train and orthodict.sbo.sbo_train is shim.sbo_train
    assert orthodict.sbo.worst_set is shim.worst_set
    shim.uninstall()
    assert orthodict.cli.sbo_train is orthodict.sbo.sbo_train
    assert orthodict.cli.sbo_train.__module__ == "orthodict.sbo"
    shim.install()


def test_result_types_are_the_references():
    import paper_1412_4944_b200 as b
    rng = np.random.default_rng(0)
    q = np.linalg.qr(rng.standard_normal((4, 4)))[0]
    d = shim.to_ref_dictionary(b.UnionDictionary([q, q]))
    assert type(d) is orthodict.sbo.UnionDictionary and d.num_blocks == 2
    code = b.SparseCode(np.zeros(3, np.int64), np.zeros((2, 3), np.int64), np.ones((2, 3)),
                        np.ones(3), np.zeros(3))
    rc = shim.to_ref_code(code)
    assert type(rc) is orthodict.sbo.SparseCode
    rep = b.TrainReport("sbo", {"s0": 2}, 0, 1, [b.IterationStats(0, 2, 0.5, 0.1, 0.2)],
                        notes=["x"])
    rr = shim.to_ref_report(rep)
    assert type(rr) is orthodict.report.TrainReport and rr.to_dict() == rep.to_dict()
    cfg = orthodict.SboConfig(s0=3, k0=2, k_max=5, energy_kind="abs-sum", seed=9)
    assert shim.to_b200_config(cfg) == b.SboConfig(s0=3, k0=2, k_max=5, energy_kind="abs-sum",
                                                   seed=9)


def test_errors_map_to_the_references_exit_codes(installed, tmp_path, monkeypatch):
    """Our NumericalError / DecompositionError reach cli.py:359 as the reference's
    classes (exit 3); ValueError stays a usage error (exit 2)."""
    import paper_1412_4944_b200 as b
    y = np.random.default_rng(1).standard_normal((4, 50))
    sig = tmp_path / "y.odm"
    orthodict.data.save_matrix(sig, y)
    for exc, code in ((b.DecompositionError("SVD did not converge for a 4x4 matrix"), 3),
                      (b.NumericalError("defect"), 3), (ValueError("bad"), 2)):
        def boom(*a, _e=exc, **k):
            raise _e
        monkeypatch.setattr(b, "sbo_train", boom)
        rc = orthodict.cli.main(["train", "--signals", str(sig), "--k0", "1", "--kmax", "2",
                                 "--out", str(tmp_path / "o")])
        assert rc == code


# ------------------------------------------------------------ the device path
gpu = pytest.mark.gpu


@gpu
def test_cli_train_and_represent_through_the_shim(installed, tmp_path, desk_y64):
    """orthodict's own CLI, unchanged, on the device path: exit 0, and the files its
    store writes from our results are byte-identical to our drop-in's own store
    writing the same results (and the report says the same)."""
    import json

    import paper_1412_4944_b200 as b
    from paper_1412_4944_b200 import store as ours
    y = desk_y64[:, :4096]
    sig = tmp_path / "y.odm"
    orthodict.data.save_matrix(sig, y)
    out = tmp_path / "train"
    rc = orthodict.cli.main(["train", "--signals", str(sig), "--k0", "3", "--kmax", "6",
                             "--r", "3", "--save-codes", "--out", str(out)])
    assert rc == 0
    d, code, a, rep = b.sbo_train(y, b.SboConfig(s0=8, k0=3, k_max=6, rounds=3, seed=0))
    mine = tmp_path / "mine"
    ours.save_dictionary(mine, d, extra_meta={"algo": "sbo", "s0": 8,
                                              "energy_kind": "squared-sum", "seed": 0})
    ours.save_sbo_codes(mine, code)
    for f in (orthodict.store.DICT_FILE, orthodict.store.DICT_META_FILE,
              orthodict.store.CODES_FILE, orthodict.store.CODES_META_FILE):
        assert (out / f).read_bytes() == (mine / f).read_bytes(), f
    got = json.loads((out / orthodict.store.REPORT_FILE).read_text())
    assert [r["rmse"] for r in got["rows"]] == [r.rmse for r in rep.rows]
    assert got["notes"] == rep.notes
    # represent with the saved dictionary
    rout = tmp_path / "rep"
    rc = orthodict.cli.main(["represent", "--signals", str(sig), "--dict", str(out),
                             "--save-codes", "--out", str(rout)])
    assert rc == 0
    a2, c2 = b.represent(y, d, 8)
    sc = b.SparseCode(a2.block, c2.indices, c2.values, a2.energy, a2.residual_sq)
    mine2 = tmp_path / "mine2"
    ours.save_sbo_codes(mine2, sc)
    assert (rout / orthodict.store.CODES_FILE).read_bytes() == \
        (mine2 / orthodict.store.CODES_FILE).read_bytes()
    res = json.loads((rout / "represent.json").read_text())
    want = b.frobenius_error(y, d, sc) / np.sqrt(y.size)
    assert res["rmse"] == pytest.approx(want, rel=1e-12)


@gpu
def test_cli_exit_3_on_injected_nonconvergence(installed, tmp_path, desk_y64, monkeypatch):
    """A device status word set to ST_NOCONV (injected into the polar status the
    retrain writes) surfaces as the reference's DecompositionError naming the
    matrix dimensions, and the reference CLI exits 3 (cli.py:359-361)."""
    from paper_1412_4944_b200 import _lib as L
    from paper_1412_4944_b200.engine import Engine
    orig = Engine.train_rounds

    def faulty(self, order, g, n, rounds, nblocks, first_block, counts, status, single):
        orig(self, order, g, n, rounds, nblocks, first_block, counts, status, single)
        status[0].fill_(L.ST_NOCONV)

    monkeypatch.setattr(Engine, "train_rounds", faulty)
    sig = tmp_path / "y.odm"
    orthodict.data.save_matrix(sig, desk_y64[:, :2048])
    with pytest.raises(orthodict.linalg.DecompositionError, match="64x64"):
        shim.sbo_train(desk_y64[:, :2048], orthodict.SboConfig(s0=8, k0=2, k_max=3, rounds=2))
    rc = orthodict.cli.main(["train", "--signals", str(sig), "--k0", "2", "--kmax", "3",
                             "--r", "2", "--out", str(tmp_path / "o")])
    assert rc == 3
