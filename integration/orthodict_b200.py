"""Reference-side binding: route ``orthodict``'s SBO entry points through the B200 path.

This is the shim a maintainer of the reference would add (e.g. as
``orthodict/_b200.py``, or imported before ``orthodict.cli``).  It is NOT part
of the product package: ``paper_1412_4944_b200`` never imports ``orthodict``.

``install()`` rebinds the names the reference binds at import time
(cli.py:32-40 ``from .sbo import ... represent, sbo_train``; the package
namespace __init__.py:30-41; sbo.py's module globals) to wrappers that

  * convert the reference's argument types to ours (``SboConfig``,
    ``UnionDictionary``, ``SparseCode``; same fields, sbo.py:34-118);
  * call the device implementation;
  * convert the results back to the reference's own classes, so that
    ``orthodict.store.save_dictionary`` (store.py:57 ``isinstance(...,
    UnionDictionary)``), ``store.save_sbo_codes`` and ``TrainReport.save``
    accept them;
  * re-raise our ``NumericalError`` / ``DecompositionError`` as the reference's
    classes (onb.py:20, linalg.py:15), which cli.py:29-30 bound at import and
    cli.py:359 maps to exit code 3.

``uninstall()`` restores the original bindings.
"""
from __future__ import annotations

import dataclasses
import functools

import numpy as np

_SAVED: list[tuple[object, str, object]] = []


def _ref():
    import orthodict
    import orthodict.cli
    import orthodict.linalg
    import orthodict.onb
    import orthodict.report
    import orthodict.sbo
    return orthodict


def _b200():
    import paper_1412_4944_b200 as b
    return b


# ------------------------------------------------------------------ conversions
def to_b200_config(cfg):
    b = _b200()
    return b.SboConfig(**dataclasses.asdict(cfg))


def to_b200_dictionary(d):
    b = _b200()
    return b.UnionDictionary([np.asarray(q, dtype=np.float64) for q in d.blocks])


def to_b200_code(code):
    b = _b200()
    return b.SparseCode(block=np.asarray(code.block), indices=np.asarray(code.indices),
                        values=np.asarray(code.values), energy=np.asarray(code.energy),
                        residual_sq=np.asarray(code.residual_sq))


def to_ref_dictionary(d):
    R = _ref()
    return R.sbo.UnionDictionary([np.asarray(q) for q in d.blocks])


def to_ref_code(code):
    R = _ref()
    return R.sbo.SparseCode(block=code.block, indices=code.indices, values=code.values,
                            energy=code.energy, residual_sq=code.residual_sq)


def to_ref_assignment(a):
    R = _ref()
    return R.sbo.Assignment(block=a.block, energy=a.energy, residual_sq=a.residual_sq)


def to_ref_thresholded(c):
    R = _ref()
    return R.onb.ThresholdedCode(indices=c.indices, values=c.values)


def to_ref_report(rep):
    R = _ref()
    return R.report.TrainReport.from_dict(rep.to_dict())


def _mapped_errors(fn):
    """Re-raise the device path's numerical exceptions as the reference's classes."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        b, R = _b200(), _ref()
        try:
            return fn(*args, **kwargs)
        except b.NumericalError as exc:
            raise R.onb.NumericalError(str(exc)) from exc
        except b.DecompositionError as exc:
            raise R.linalg.DecompositionError(str(exc)) from exc

    return wrapper


# --------------------------------------------------------------------- wrappers
@_mapped_errors
def sbo_train(y, cfg, workers=None):
    """orthodict.sbo_train (sbo.py:299-420) on the device; reference result types."""
    d, code, a, rep = _b200().sbo_train(y, to_b200_config(cfg), workers=workers)
    return to_ref_dictionary(d), to_ref_code(code), to_ref_assignment(a), to_ref_report(rep)


@_mapped_errors
def represent(y, dictionary, s0, kind="squared-sum", chunk_size=256, workers=None):
    """orthodict.represent (sbo.py:138-220) on the device; reference result types."""
    a, c = _b200().represent(y, to_b200_dictionary(dictionary), s0, kind, chunk_size, workers)
    return to_ref_assignment(a), to_ref_thresholded(c)


@_mapped_errors
def sbo_init(y, cfg, workers=None):
    """orthodict.sbo.sbo_init (sbo.py:259-292) on the device."""
    return to_ref_dictionary(_b200().sbo_init(y, to_b200_config(cfg), workers=workers))


@_mapped_errors
def worst_set(assignment, w):
    return _b200().worst_set(assignment, w)


@_mapped_errors
def group_by_block(y, assignment, num_blocks=None):
    return _b200().group_by_block(y, assignment, num_blocks)


@_mapped_errors
def frobenius_error(y, dictionary, code):
    """linalg.py:89-102 for the SBO pairing (union + single-best-block code) on the
    device; any other pairing goes to the reference's own function."""
    R = _ref()
    if isinstance(dictionary, R.sbo.UnionDictionary) and isinstance(code, R.sbo.SparseCode):
        return _b200().frobenius_error(y, to_b200_dictionary(dictionary), to_b200_code(code))
    return _ORIGINAL["frobenius_error"](y, dictionary, code)


_ORIGINAL: dict[str, object] = {}

# (module attribute path, wrapper) pairs; each name is rebound wherever the
# reference bound it at import time
_BINDINGS = {
    "sbo_train": ("orthodict", "orthodict.sbo", "orthodict.cli"),
    "represent": ("orthodict", "orthodict.sbo", "orthodict.cli"),
    "sbo_init": ("orthodict", "orthodict.sbo"),
    "worst_set": ("orthodict", "orthodict.sbo"),
    "group_by_block": ("orthodict", "orthodict.sbo"),
    "frobenius_error": ("orthodict", "orthodict.linalg", "orthodict.cli"),
}


def install() -> None:
    """Rebind orthodict's SBO entry points to the device path (idempotent)."""
    import importlib
    if _SAVED:
        return
    _ref()
    wrappers = globals()
    for name, modules in _BINDINGS.items():
        for modname in modules:
            mod = importlib.import_module(modname)
            orig = getattr(mod, name)
            _ORIGINAL.setdefault(name, orig)
            _SAVED.append((mod, name, orig))
            setattr(mod, name, wrappers[name])


def uninstall() -> None:
    """Restore the reference's own bindings."""
    while _SAVED:
        mod, name, orig = _SAVED.pop()
        setattr(mod, name, orig)
    _ORIGINAL.clear()
