"""ctypes binding of the C ABI (include/sbo_b200.h) — the only way into the kernels.

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
next to this file.  There is no fallback: if the library or a CUDA device is
missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# SBO_LIB: an alternative in-tree build of the same library (A/B measurements)
LIB_PATH = Path(__file__).resolve().parent / os.environ.get("SBO_LIB", "libsbo_b200.so")

OK, EINVAL, ENUMERICAL, EDECOMP, ECUDA = 0, 1, 2, 3, 4
KIND = {"squared-sum": 0, "abs-sum": 1}
F32, F64 = 0, 1
ST_OK, ST_SKIPPED, ST_DEFECT, ST_NOCONV = 0, 1, 2, 3

P, I, I64, SZ, D = C.c_void_p, C.c_int, C.c_int64, C.c_size_t, C.c_double

# name -> (restype, argtypes); mirrors include/sbo_b200.h
_SIGS = {
    "sbo_abi_version": (I, []),
    "sbo_last_error": (C.c_char_p, []),
    "sbo_device_ok": (I, [I]),
    "sbo_energy_pass": (I, [P, I, I64, I, P, I, I, I, I, I, P, P, P, P, P]),
    "sbo_energy_recheck": (I, [P, I, I64, I, P, I, I, I, I, P, P, I64, P, P, P, P]),
    "sbo_tc_padded_rows": (I64, [I64]),
    "sbo_tc_split_signals": (I, [P, I, I64, I, P, P, P, P]),
    "sbo_tc_split_blocks": (I, [P, I, I, P, P, P, P]),
    "sbo_tc_energy": (I, [P, P, P, I64, P, P, P, I, I, I, I, I, P, P, P, P, P, P, P]),
    "sbo_tc_energy256": (I, [P, P, P, I64, P, P, P, I, I, I, I, I, P, P, P, P, P, P, P]),
    "sbo_cand_workspace_bytes": (SZ, []),
    "sbo_cand_sort": (I, [P, P, P, I64, P, P, P, SZ, P]),
    "sbo_energy_recheck_cand": (I, [P, I, I64, I, P, I, I, I, P, P, P, I64, P, P, P, P]),
    "sbo_group_workspace_bytes": (SZ, [I64, I]),
    "sbo_max_segments": (I64, [I64, I, I]),
    "sbo_group": (I, [P, I64, I, I, P, P, P, P, P, P, P, SZ, P]),
    "sbo_code_segments": (I, [P, I, I, P, P, P, P, P, I64, P, I, I, I, I, I64, P, P, P, P, P]),
    "sbo_outer_segments": (I, [P, I, I, P, P, P, P, I64, I, I64, P, P, P, P]),
    "sbo_reduce_segments": (I, [P, P, P, I64, I, I, P, P]),
    "sbo_round_segments": (I, [P, I, I, P, P, P, P, P, I64, P, I, I, P, P]),
    "sbo_residual_segments": (I, [P, I, I, P, P, P, P, P, I64, P, I, I, P, P, P]),
    "sbo_round_code_segments": (I, [P, I, I, P, P, P, P, P, I64, P, I, I, I64, P, P, P]),
    "sbo_outer_i8_segments": (I, [P, I, P, P, P, P, I64, I, I, I64, P, P, I, I, P, P, SZ, P]),
    "sbo_round_i8_workspace_bytes": (SZ, [I]),
    "sbo_round_i8_segments": (I, [P, I, P, P, P, P, P, I64, P, I, I, I, I, I, I64, P, P, P, P,
                                  P, SZ, P]),
    "sbo_y_tiles_bytes": (SZ, [I64, I64, I]),
    "sbo_y_tiles": (I, [P, I, P, P, P, P, I64, P, P]),
    "sbo_outer_i8_workspace_bytes": (SZ, [I, I]),
    "sbo_i8_scan": (I, [P, I, I64, I, P, P]),
    "sbo_y_digits": (I, [P, I, I64, I, I, P, P]),
    "sbo_gram_workspace_bytes": (SZ, [I64, I, I]),
    "sbo_gram": (I, [P, I, I, P, I64, I, P, P, SZ, P]),
    "sbo_gram_counted": (I, [P, I, I, P, I64, P, I, P, P, SZ, P]),
    "sbo_chunk_segments": (I, [I64, P, I, P, P, P, P]),
    "sbo_select_top": (I, [P, I64, I, I, I64, P, P, P]),
    "sbo_select_coded": (I, [P, P, I64, I, I, I, P, I64, P, P, P, P, P]),
    "sbo_coef_i8_workspace_bytes": (SZ, [I]),
    "sbo_coef_i8_segments": (I, [P, I, P, P, P, P, P, I64, P, I, I, P, P, SZ, P]),
    "sbo_recheck_i8_workspace_bytes": (SZ, [I]),
    "sbo_recheck_pairs_workspace_bytes": (SZ, [I, I64]),
    "sbo_energy_recheck_pairs": (I, [P, I, P, I, I, I, P, P, P, I64, P, P, P, P, SZ, P]),
    "sbo_energy_recheck_i8": (I, [P, I, P, I, I, I, P, P, P, I64, P, P, P, P, SZ, P]),
    "sbo_polar_workspace_bytes": (SZ, [I, I]),
    "sbo_polar": (I, [P, I, I, P, P, P, P, P, P, SZ, P]),
    "sbo_init_workspace_bytes": (SZ, [I]),
    "sbo_init_block": (I, [P, I, I64, P, I, P, P, P, P, SZ, P]),
    "sbo_svd_workspace_bytes": (SZ, [I, I]),
    "sbo_svd": (I, [P, I, I, P, P, P, P, P, SZ, P]),
    "sbo_worst_workspace_bytes": (SZ, [I64]),
    "sbo_worst_set": (I, [P, I64, I64, P, P, SZ, P]),
    "sbo_key_histogram": (I, [P, I64, C.c_uint64, I, P, P]),
    "sbo_worst_collect": (I, [P, I64, C.c_uint64, I64, P, P, P, SZ, P]),
    "sbo_select_begin": (I, [P, I64, P]),
    "sbo_select_hist": (I, [P, I64, P, I, P, P]),
    "sbo_select_pick": (I, [P, P, I, P]),
    "sbo_select_counts": (I, [P, I64, P, SZ, P, P]),
    "sbo_select_write": (I, [P, I64, P, SZ, P, P, I, P, P, P]),
    "sbo_sum_workspace_bytes": (SZ, [I64]),
    "sbo_sum": (I, [P, I64, P, P, SZ, P]),
    "sbo_defect": (I, [P, I, I, P, P]),
    "sbo_frobenius_sq": (I, [P, I, I64, I, P, P, I, I64, P, P, P, P, SZ, P]),
    "sbo_extract_patches": (I, [P, I, I64, I64, I64, I, P, P, I64, I, I, P, P]),
    "sbo_codes_pack": (I, [I, P, P, P, I64, I, I64, I64, P, P]),
}

_lib = None


class KernelLibraryMissing(RuntimeError):
    """The in-tree CUDA library is absent (build it with ``make``)."""


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise KernelLibraryMissing(
                f"{LIB_PATH} not found: build the sm_100a library (make, or __graft_entry__.build())")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(h, name)
            f.restype, f.argtypes = res, args
        _lib = h
    return _lib


def exported_symbols():
    return list(_SIGS)


def _raise(code: int, where: str):
    from .linalg import DecompositionError
    from .onb import NumericalError
    msg = f"{where}: {lib().sbo_last_error().decode(errors='replace')}"
    if code == EINVAL:
        raise ValueError(msg)
    if code == ENUMERICAL:
        raise NumericalError(msg)
    if code == EDECOMP:
        raise DecompositionError(msg)
    raise RuntimeError(msg)


def call(name: str, *args):
    """Invoke an ABI entry point; map a nonzero status onto the reference's exceptions."""
    rc = getattr(lib(), name)(*args)
    if rc != OK:
        _raise(rc, name)
    return rc


def size(name: str, *args) -> int:
    return int(getattr(lib(), name)(*args))


def debug_sync() -> bool:
    return os.environ.get("SBO_DEBUG_SYNC", "0") == "1"
