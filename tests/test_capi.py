"""The C-ABI library loads and exports every symbol include/sbo_b200.h declares (CPU)."""
import ctypes
import re

from conftest import REPO
from paper_1412_4944_b200 import _lib


def declared_functions():
    text = (REPO / "include" / "sbo_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sbo_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_lib.exported_symbols())


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_host_side_queries_without_gpu():
    lib = _lib.lib()
    assert lib.sbo_abi_version() == 1
    assert lib.sbo_max_segments(1 << 20, 16, 1024) == 1024 + 16
    assert lib.sbo_group_workspace_bytes(1 << 20, 16) > 0
    assert lib.sbo_worst_workspace_bytes(1 << 20) > 0
    assert lib.sbo_polar_workspace_bytes(16, 64) >= 16 * 2 * 64 * 64 * 8


def test_invalid_arguments_are_rejected_before_launch():
    lib = _lib.lib()
    # p out of range and bad dtype fail argument validation on the host side
    rc = lib.sbo_energy_pass(None, 0, 10, 300, None, 0, 1, 8, 0, 0, None, None, None, None, None)
    assert rc == _lib.EINVAL
    assert b"p must be" in lib.sbo_last_error()
    rc = lib.sbo_energy_pass(None, 7, 10, 64, None, 0, 1, 8, 0, 0, None, None, None, None, None)
    assert rc == _lib.EINVAL


def test_product_package_never_imports_the_oracle():
    pat = re.compile(r"^\s*(from|import)\s+oracle\b", re.M)
    for path in (REPO / "paper_1412_4944_b200").rglob("*.py"):
        assert not pat.search(path.read_text()), path
