"""Artifact storage: byte-identical to the reference's store.py
(golden files written by the real reference), and device-streamed codes identical
to the host writer."""
from pathlib import Path

import numpy as np
import pytest

from conftest import golden, has_cuda
from paper_1412_4944_b200 import store
from paper_1412_4944_b200.sbo import SparseCode, UnionDictionary


def _code(g):
    return SparseCode(g["block"], g["indices"], g["values"], g["energy"], g["residual_sq"])


def test_codes_files_match_reference(tmp_path):
    g = golden("store_files")
    store.save_sbo_codes(tmp_path, _code(g))
    assert (tmp_path / "codes.odm").read_bytes() == g["codes_odm"].tobytes()
    assert (tmp_path / "codes.meta.json").read_text() == str(g["codes_meta"])
    back = store.load_sbo_codes(tmp_path)
    for name in ("block", "indices", "values", "energy", "residual_sq"):
        np.testing.assert_array_equal(getattr(back, name), g[name])


def test_dictionary_files_match_reference(tmp_path):
    g = golden("store_files")
    store.save_dictionary(tmp_path / "u", UnionDictionary(list(g["union"])), {"note": "x"})
    assert (tmp_path / "u" / "dict.odm").read_bytes() == g["union_odm"].tobytes()
    assert (tmp_path / "u" / "dict.meta.json").read_text() == str(g["union_meta"])
    d, header = store.load_dictionary(tmp_path / "u")
    assert header["format"] == "union-onb" and header["note"] == "x"
    np.testing.assert_array_equal(np.stack(d.blocks), g["union"])
    store.save_dictionary(tmp_path / "d", g["dense"])
    assert (tmp_path / "d" / "dict.odm").read_bytes() == g["dense_odm"].tobytes()
    assert (tmp_path / "d" / "dict.meta.json").read_text() == str(g["dense_meta"])
    dense, header = store.load_dictionary(tmp_path / "d")
    assert header == {"format": "dense", "p": 6, "atoms": 9}
    np.testing.assert_array_equal(dense, g["dense"])


def test_record_errors(tmp_path):
    with pytest.raises(store.MatrixFormatError, match="bad magic"):
        store.read_record(b"XXXX" + bytes(16), 0)
    with pytest.raises(store.MatrixFormatError, match="truncated header"):
        store.read_record(b"ODM1" + bytes(8), 0)
    with pytest.raises(store.MatrixFormatError, match="truncated payload"):
        store.read_record(b"ODM1" + store.ODM_HEADER.pack(2, 2) + bytes(8), 0)
    with pytest.raises(ValueError, match="ODM1 stores 2-D matrices"):
        with open(tmp_path / "x", "wb") as f:
            store.write_record(f, np.zeros(3))
    (tmp_path / "codes.meta.json").write_text('{"format": "other"}\n')
    with pytest.raises(store.MatrixFormatError, match="not an sbo codes file"):
        store.load_sbo_codes(tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [7, 1 << 20])
def test_device_codes_stream_identical_bytes(tmp_path, chunk):
    import paper_1412_4944_b200 as S
    from paper_1412_4944_b200 import data, signals
    grid = signals.scene(128, 128, 1)
    y = data.extract_patches(grid, data.PatchConfig(patch_edge=8, count=1500, seed=2))
    rng = np.random.default_rng(3)
    d = S.UnionDictionary([np.linalg.qr(rng.standard_normal((64, 64)))[0] for _ in range(4)])
    dc = S.represent_device(y, d, 8)
    store.save_sbo_codes(tmp_path / "dev", dc, chunk=chunk)
    a, code = S.represent(y, d, 8)
    host = SparseCode(a.block, code.indices, code.values, a.energy, a.residual_sq)
    store.save_sbo_codes(tmp_path / "host", host)
    for name in ("codes.odm", "codes.meta.json"):
        assert (tmp_path / "dev" / name).read_bytes() == (tmp_path / "host" / name).read_bytes()
    back = store.load_sbo_codes(tmp_path / "dev")
    np.testing.assert_array_equal(back.block, a.block)
    np.testing.assert_array_equal(back.values, code.values)
