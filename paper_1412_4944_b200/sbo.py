"""Single-Block-Orthogonal dictionary learning on the device (mirror of orthodict.sbo).

Drop-in for the reference's SBO entry points (sbo.py:34-436): same types,
names, argument meaning, tie rules, note strings and exceptions.  The signal
matrix is uploaded once per call and everything numeric runs in the sm_100a
library (see engine.py for the kernel sequence of one iteration).

Signals are held as float32 on the device when that is exact (every value
float32-representable — the benchmark's image patches), otherwise as float64.
``workers`` and ``chunk_size`` are validated like the reference and, as there,
never change results.
"""
from __future__ import annotations

import math
import warnings
from dataclasses import dataclass
from time import perf_counter

import numpy as np
import torch

from . import _lib as L
from .engine import Comm, Engine, Signals, check_status, require_device
from .onb import ThresholdedCode
from .parallel import resolve_workers
from .report import IterationStats, TrainReport

REPRESENT_TILE = 256  # sbo.py:28-29 (the reference's arithmetic tile; ours is the CUDA tile)
ENERGY_KINDS = ("squared-sum", "abs-sum")  # sbo.py:31


@dataclass
class UnionDictionary:
    """Ordered union of p x p orthonormal blocks (sbo.py:34-58)."""

    blocks: list

    @property
    def p(self) -> int:
        return self.blocks[0].shape[0]

    @property
    def num_blocks(self) -> int:
        return len(self.blocks)

    def stacked(self) -> np.ndarray:
        return np.hstack(self.blocks)

    def validate(self) -> None:
        if not self.blocks:
            raise ValueError("a union dictionary needs at least one block")
        p = self.p
        for i, q in enumerate(self.blocks):
            if q.shape != (p, p):
                raise ValueError(f"block {i} has shape {q.shape}, expected ({p}, {p})")


@dataclass
class Assignment:
    """Per-signal best block, its energy and the squared residual (sbo.py:61-67)."""

    block: np.ndarray
    energy: np.ndarray
    residual_sq: np.ndarray


@dataclass
class SparseCode:
    """Single-best-block sparse representation (sbo.py:70-78)."""

    block: np.ndarray
    indices: np.ndarray
    values: np.ndarray
    energy: np.ndarray
    residual_sq: np.ndarray


@dataclass
class SboConfig:
    """Training knobs (sbo.py:81-118); worst_size defaults to max(p, m // 16)."""

    s0: int
    k0: int = 5
    p0: int = 4096
    rounds: int = 6
    worst_size: int | None = None
    k_max: int = 64
    target_error: float = 0.0
    energy_kind: str = "squared-sum"
    seed: int = 0
    chunk_size: int = REPRESENT_TILE

    def validate(self) -> None:
        checks = (
            (self.s0 < 1, f"s0 must be at least 1, got {self.s0}"),
            (self.k0 < 1, f"k0 must be at least 1, got {self.k0}"),
            (self.p0 < 1, f"p0 must be at least 1, got {self.p0}"),
            (self.rounds < 0, f"rounds must be nonnegative, got {self.rounds}"),
            (self.k0 > self.k_max, f"k0 ({self.k0}) exceeds k_max ({self.k_max})"),
            (self.chunk_size < 1, f"chunk_size must be at least 1, got {self.chunk_size}"),
            (self.worst_size is not None and self.worst_size < 1,
             f"worst_size must be at least 1, got {self.worst_size}"),
            (self.target_error < 0, f"target_error must be nonnegative, got {self.target_error}"),
        )
        for bad, msg in checks:
            if bad:
                raise ValueError(msg)
        _check_kind(self.energy_kind)


def _check_kind(kind: str) -> None:
    if kind not in ENERGY_KINDS:
        raise ValueError(f"energy_kind must be one of {ENERGY_KINDS}, got {kind!r}")


def _block_rng(seed: int, phase: int, ordinal: int) -> np.random.Generator:
    """sbo.py:252-256 — independent stream per (phase, block ordinal)."""
    entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF, phase, ordinal]
    return np.random.default_rng(np.random.SeedSequence(entropy))


def _device_signals(y) -> tuple[Signals, int, int]:
    """Signals already on the device (data.extract_patches_device): validated there."""
    if not torch.isfinite(y.y).all().item():
        raise ValueError("signal matrix contains NaN or Inf entries")
    return y, y.p, y.m


def _signals(y, dev) -> tuple[Signals, int, int]:
    """(device signals, p, m) from a host p x m matrix or device Signals."""
    if isinstance(y, Signals):
        return _device_signals(y)
    y = _check_signals(y)
    return Signals.from_reference(y, dev), y.shape[0], y.shape[1]


def _check_signals(y) -> np.ndarray:
    y = np.asarray(y, dtype=np.float64)
    if y.ndim != 2:
        raise ValueError(f"expected a 2-D signal matrix, got shape {y.shape}")
    if not np.isfinite(y).all():
        raise ValueError("signal matrix contains NaN or Inf entries")
    return y


# ---------------------------------------------------------------------------
# representation
# ---------------------------------------------------------------------------

def block_energy(y: np.ndarray, q: np.ndarray, s0: int, kind: str = "squared-sum") -> float:
    """sbo.py:126-135 — hard-thresholded energy of one signal in one block."""
    _check_kind(kind)
    y = np.asarray(y, dtype=np.float64).ravel()
    q = np.asarray(q, dtype=np.float64)
    # the exact float64 energy pass (the tensor-core pass's score is only
    # float32-accurate; it certifies decisions, not values)
    eng = Engine(Signals.from_reference(y[:, None], require_device()), s0, kind, k_cap=1,
                 tc=False)
    eng.set_blocks(q[None])
    eng.energy(0, 1, False)
    return float(eng.state.score[0].item())


def _code_all(eng: Engine):
    """Both passes of represent on an engine: returns device (best, energy, residual, idx, val)."""
    m, K = eng.m, eng.K
    eng.energy(0, K, False)
    g = eng.group(K)
    energy = torch.empty(m, dtype=torch.float64, device=eng.dev)
    idx = torch.empty((eng.k, max(m, 1)), dtype=torch.int16, device=eng.dev)
    val = torch.empty((eng.k, max(m, 1)), dtype=torch.float64, device=eng.dev)
    # pass 2 codes each winner with its block; kept sums come from the kept values
    eng.code(g.perm, g, -1, True, m, idx, val, energy, eng.state.residual)
    eng.residual()
    return eng.state.best, energy, eng.state.residual, idx, val


def represent(y: np.ndarray, dictionary: UnionDictionary, s0: int, kind: str = "squared-sum",
              chunk_size: int = REPRESENT_TILE, workers: int | None = None
              ) -> tuple[Assignment, ThresholdedCode]:
    """sbo.py:138-220 — best block per signal (first maximum) and its top-s0 code."""
    _check_kind(kind)
    dictionary.validate()
    dev = require_device()
    sig, p, m = _signals(y, dev)
    if p != dictionary.p:
        raise ValueError(f"signals have dimension {p}, dictionary blocks {dictionary.p}")
    if s0 < 1:
        raise ValueError(f"s0 must be at least 1, got {s0}")
    if chunk_size < 1:
        raise ValueError(f"chunk_size must be at least 1, got {chunk_size}")
    resolve_workers(workers)
    eng = Engine(sig, s0, kind, k_cap=dictionary.num_blocks)
    eng.set_blocks(np.stack(dictionary.blocks))
    best, energy, resid, idx, val = _code_all(eng)
    k = eng.k
    return (Assignment(best.cpu().numpy().astype(np.int64), energy.cpu().numpy(),
                       resid.cpu().numpy()),
            ThresholdedCode(idx[:, :m].cpu().numpy().astype(np.int64), val[:, :m].cpu().numpy()))


def represent_device(y, dictionary: UnionDictionary, s0: int, kind: str = "squared-sum",
                     chunk_size: int = REPRESENT_TILE, workers: int | None = None):
    """represent() with the result left on the device: a ``store.DeviceCode`` (for
    streaming to disk with ``store.save_sbo_codes`` or further device work).  Same
    validation and values as represent()."""
    from .store import DeviceCode
    _check_kind(kind)
    dictionary.validate()
    dev = require_device()
    sig, p, m = _signals(y, dev)
    if p != dictionary.p:
        raise ValueError(f"signals have dimension {p}, dictionary blocks {dictionary.p}")
    if s0 < 1:
        raise ValueError(f"s0 must be at least 1, got {s0}")
    if chunk_size < 1:
        raise ValueError(f"chunk_size must be at least 1, got {chunk_size}")
    resolve_workers(workers)
    eng = Engine(sig, s0, kind, k_cap=dictionary.num_blocks)
    eng.set_blocks(np.stack(dictionary.blocks))
    best, energy, resid, idx, val = _code_all(eng)
    return DeviceCode(best, idx, val, energy, resid)


def worst_set(assignment: Assignment, w: int) -> np.ndarray:
    """sbo.py:223-228 — the w largest residuals, descending, ties toward low indices."""
    if w < 1:
        raise ValueError(f"worst-set size must be at least 1, got {w}")
    res = np.asarray(assignment.residual_sq, dtype=np.float64)
    m = res.shape[0]
    if m == 0:
        return np.empty(0, np.int64)
    dev = require_device()
    r = torch.from_numpy(np.ascontiguousarray(res)).to(dev)
    n = min(w, m)
    members = torch.empty(n, dtype=torch.int32, device=dev)
    ws = torch.empty(L.size("sbo_worst_workspace_bytes", m), dtype=torch.uint8, device=dev)
    L.call("sbo_worst_set", r.data_ptr(), m, w, members.data_ptr(), ws.data_ptr(), ws.numel(),
           torch.cuda.current_stream(dev).cuda_stream)
    # the set is what training consumes; the reference also returns it sorted
    # by descending residual (stable, so ties keep ascending index order)
    order = torch.sort(-r[members.long()], stable=True).indices
    return members.long()[order].cpu().numpy()


def group_by_block(y: np.ndarray, assignment: Assignment, num_blocks: int | None = None
                   ) -> tuple[np.ndarray, list[tuple[int, int]], np.ndarray]:
    """sbo.py:231-249 — stable permutation by block, per-block ranges, permuted signals."""
    block = np.asarray(assignment.block)
    if num_blocks is None:
        num_blocks = int(block.max()) + 1 if block.size else 0
    m = block.shape[0]
    # the counting sort runs on the device over ids shifted to start at 0 (a
    # stable sort by id is invariant under the shift), so negative ids order
    # first, as numpy's argsort puts them
    lo = int(block.min()) if m else 0
    shift = min(lo, 0)
    K = max(num_blocks - shift, int(block.max()) - shift + 1 if m else 0, 1)
    dev = require_device()
    eng = Engine(Signals(torch.zeros((max(m, 1), 1), dtype=torch.float64, device=dev)), 1,
                 k_cap=1)
    eng.m = m
    eng.state.best = torch.from_numpy((block.astype(np.int64) - shift).astype(np.int32)).to(dev)
    g = eng.group(K)
    perm = g.perm[:m].long().cpu().numpy()
    bounds = g.bounds.cpu().numpy()
    ranges = [(int(bounds[b - shift]), int(bounds[b - shift + 1])) for b in range(num_blocks)]
    # the permuted matrix in the caller's dtype, like the reference's y[:, perm]
    grouped = np.asarray(y)[:, perm]
    return grouped, ranges, perm


# ---------------------------------------------------------------------------
# training
# ---------------------------------------------------------------------------

def _init_into(eng: Engine, cfg: SboConfig, m_total: int, local_cols=None) -> None:
    """sbo.py:259-292 on the device: block b from p0 seeded samples -> init -> R rounds.

    ``local_cols(cols)`` maps global sample columns to this shard's local member
    list (multi-GPU); None means the engine holds every signal."""
    p = eng.p
    replace = cfg.p0 > m_total
    eng.ensure_capacity(cfg.k0)
    st = torch.zeros((cfg.k0, cfg.rounds + 1, 1), dtype=torch.int32, device=eng.dev)
    for b in range(cfg.k0):
        rng = _block_rng(cfg.seed, 0, b)
        cols = rng.choice(m_total, size=cfg.p0, replace=replace)
        draws = rng.standard_normal((p + 8, p))
        members = cols if local_cols is None else local_cols(cols)
        mem = torch.from_numpy(members.astype(np.int32)).to(eng.dev)
        n = int(members.shape[0])
        G = eng.comm.allreduce(eng.gram(mem, n))
        eng.init_block(G, cfg.p0, draws, b, st[b, cfg.rounds])
        eng.train_rounds(mem, eng.list_segments(n), n, cfg.rounds, 1, b, None, st[b],
                         single=True)
    eng.K = cfg.k0
    check_status(st.cpu().numpy(), p)


def sbo_init(y: np.ndarray, cfg: SboConfig, workers: int | None = None) -> UnionDictionary:
    """sbo.py:259-292 — k0 start-up blocks, each trained on p0 sampled signals."""
    cfg.validate()
    if not isinstance(y, Signals):
        y = np.asarray(y, dtype=np.float64)
    m = y.m if isinstance(y, Signals) else y.shape[1]
    if m < 1:
        raise ValueError("cannot initialize from an empty signal set")
    if cfg.p0 > m:
        warnings.warn(f"p0={cfg.p0} exceeds the {m} available signals; sampling with "
                      "replacement", stacklevel=2)
    resolve_workers(workers)
    sig, _, _ = _signals(y, require_device())
    eng = Engine(sig, cfg.s0, cfg.energy_kind, k_cap=cfg.k0)
    _init_into(eng, cfg, m)
    return UnionDictionary([q for q in eng.blocks[: cfg.k0].cpu().numpy()])


def _config_echo(cfg: SboConfig, w_size: int) -> dict:
    return {"s0": cfg.s0, "k0": cfg.k0, "p0": cfg.p0, "rounds": cfg.rounds,
            "worst_size": w_size, "k_max": cfg.k_max, "target_error": cfg.target_error,
            "energy_kind": cfg.energy_kind, "seed": cfg.seed, "chunk_size": cfg.chunk_size}


def _rmse(assignment: Assignment, p: int, m: int) -> float:
    """sbo.py:295-296."""
    return math.sqrt(max(float(assignment.residual_sq.sum()), 0.0) / (p * m))


class _Timer:
    """CUDA-event phase timer on the engine's stream."""

    def __init__(self):
        self.ev = []

    def mark(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev.append(e)

    def spans(self):
        torch.cuda.synchronize()
        return [a.elapsed_time(b) / 1e3 for a, b in zip(self.ev, self.ev[1:])]


def train_engine(eng: Engine, cfg: SboConfig, w_size: int, report: TrainReport) -> None:
    """The sbo_train loop body on an initialized engine (sbo.py:337-397)."""
    t = _Timer()
    t.mark()
    eng.represent_full()
    t.mark()
    rmse = eng.rmse()
    report.rows.append(IterationStats(0, eng.K, rmse, report.t_init, t.spans()[0]))
    while rmse > cfg.target_error and eng.K < cfg.k_max:
        iteration = len(report.rows)
        draws = _block_rng(cfg.seed, 1, eng.K).standard_normal((eng.p + 8, eng.p))
        t = _Timer()
        out = eng.iterate(w_size, cfg.rounds, draws, timer=t)
        learn_a, rep1, learn_b, rep2 = t.spans()
        for b in out.empty_blocks:
            report.notes.append(f"iteration {iteration}: block {b} had no signals, left unchanged")
        rmse = out.rmse
        report.rows.append(IterationStats(iteration, eng.K, rmse, learn_a + learn_b, rep1 + rep2))


def sbo_train(y: np.ndarray, cfg: SboConfig, workers: int | None = None
              ) -> tuple[UnionDictionary, SparseCode, Assignment, TrainReport]:
    """sbo.py:299-420 — initialize, then grow by one block per iteration and refine,
    until the RMSE reaches target_error or the union holds k_max blocks."""
    cfg.validate()
    if isinstance(y, Signals):
        p, m = y.p, y.m
    else:
        y = np.asarray(y, dtype=np.float64)
        if y.ndim != 2:
            raise ValueError(f"expected a 2-D signal matrix, got shape {y.shape}")
        p, m = y.shape
    if m < 1:
        raise ValueError("cannot train on an empty signal set")
    nworkers = resolve_workers(workers)
    w_size = cfg.worst_size if cfg.worst_size is not None else max(p, m // 16)
    report = TrainReport(algo="sbo", config=_config_echo(cfg, w_size), seed=cfg.seed,
                         workers=nworkers)
    if cfg.p0 > m:
        report.notes.append(f"p0={cfg.p0} exceeds m={m}; initial blocks sampled with replacement")
    dev = require_device()
    sig, _, _ = _signals(y, dev)
    eng = Engine(sig, cfg.s0, cfg.energy_kind, k_cap=cfg.k_max)
    t0 = perf_counter()
    _init_into(eng, cfg, m)
    torch.cuda.synchronize(dev)
    report.t_init = perf_counter() - t0
    train_engine(eng, cfg, w_size, report)
    report.finalize_totals()
    # final timed representation with codes (sbo.py:401-407)
    t = _Timer()
    t.mark()
    best, energy, resid, idx, val = _code_all(eng)
    t.mark()
    report.t_rep = t.spans()[0]
    assignment = Assignment(best.cpu().numpy().astype(np.int64), energy.cpu().numpy(),
                            resid.cpu().numpy())
    code = SparseCode(assignment.block, idx[:, :m].cpu().numpy().astype(np.int64),
                      val[:, :m].cpu().numpy(), assignment.energy, assignment.residual_sq)
    report.rmse_final = _rmse(assignment, p, m)
    report.rmse_recomputed = math.sqrt(max(_frob_sq(eng, idx, val), 0.0) / (p * m))
    dictionary = UnionDictionary([q for q in eng.blocks[: eng.K].cpu().numpy()])
    return dictionary, code, assignment, report


def _frob_sq(eng: Engine, idx, val) -> float:
    tot = torch.zeros(1, dtype=torch.float64, device=eng.dev)
    ws = eng.scratch.get("frob", 8 * (eng.m // 8 + 2))
    eng._call("sbo_frobenius_sq", eng.sig.y.data_ptr(), eng.sig.code, eng.m, eng.p,
              eng.blocks.data_ptr(), eng.state.best.data_ptr(), eng.k, idx.shape[1],
              idx.data_ptr(), val.data_ptr(), tot.data_ptr(), ws.data_ptr(), ws.numel(),
              eng.stream)
    return float(eng.comm.allreduce(tot).item())
