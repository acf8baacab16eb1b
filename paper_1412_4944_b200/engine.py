"""Device-resident SBO engine: the host orchestration of one iteration.

Everything numeric runs in the sm_100a library through the C ABI
(include/sbo_b200.h); this module owns device buffers (allocated with torch,
which is only plumbing here: memory, streams, NCCL), sequences the kernels of
one ``sbo_train`` loop body (sbo.py:352-397) without host round-trips, and
performs the cross-rank reductions when signals are sharded over GPUs.

Per iteration (K-1 blocks entering, K leaving):
  worst set      sbo_worst_set (radix select, ties -> low index)   sbo.py:353
  new block      sbo_gram -> [allreduce] -> sbo_init_block          sbo.py:354-356
                 R x (code -> outer -> reduce -> [allreduce] -> polar)
  represent #1   sbo_energy_pass(accumulate, new block only)        sbo.py:361
  group          sbo_group (stable counting sort + segment table)  sbo.py:367
  retrain        R x (code -> outer -> reduce -> [allreduce] -> polar) sbo.py:369-385
  represent #2   sbo_energy_pass(all blocks) + sbo_residual         sbo.py:389-394
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

SEG_LEN = int(os.environ.get("SBO_SEG_LEN", 1024))  # max signals per segment of the per-block kernels
FILL_CTAS = 2 * 148   # enough segments to fill every SM twice


def seg_len(n: int) -> int:
    """Segment length (multiple of 64, <= SEG_LEN) giving ~FILL_CTAS segments for n signals."""
    want = -(-max(n, 1) // FILL_CTAS)
    return int(min(SEG_LEN, max(64, -(-want // 64) * 64)))


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


class Comm:
    """Cross-rank reductions; the single-GPU instance is the identity."""

    world = 1
    rank = 0

    def allreduce(self, t: torch.Tensor) -> torch.Tensor:
        return t

    def allgather_int(self, v: int) -> list[int]:
        return [v]

    def allgather(self, t):
        return t


class TorchComm(Comm):
    """NCCL (or gloo) process group of torch.distributed."""

    def __init__(self, group=None, sharded: bool = False):
        """``sharded=True`` runs the sharded code path (device-side worst-set select
        through the collectives) even at world size 1 — how the NCCL capture of the
        sharded step is tested on a one-GPU box."""
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.sharded = sharded
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        # NCCL collectives are stream-ordered device work (CUDA-graph capturable)
        self.capturable = dist.get_backend(group) == "nccl"

    def allreduce(self, t):
        if t.is_cuda and self.dist.get_backend(self.group) != "nccl":
            h = t.cpu()  # gloo (tests, single-GPU multi-rank runs): through the host
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
            return t
        self.dist.all_reduce(t, group=self.group)
        return t

    def allgather(self, t):
        """Concatenation over ranks of a 1-D tensor (device-resident on NCCL)."""
        if t.is_cuda and self.dist.get_backend(self.group) != "nccl":
            h = t.cpu()
            out = [torch.zeros_like(h) for _ in range(self.world)]
            self.dist.all_gather(out, h, group=self.group)
            return torch.cat(out).to(t.device)
        out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out

    def allgather_int(self, v):
        t = torch.tensor([v], dtype=torch.int64, device=_comm_device(self.dist))
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(x.item()) for x in out]


def _comm_device(dist):
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
        else torch.device("cpu")


def require_device(index: int | None = None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the SBO kernels require an sm_100a GPU (B200)")
    dev = torch.device("cuda", torch.cuda.current_device() if index is None else index)
    if not L.lib().sbo_device_ok(dev.index):
        raise RuntimeError(f"device {dev} is not an sm_100 (Blackwell) GPU")
    return dev


class Scratch:
    """Grow-only named device scratch buffers."""

    def __init__(self, device):
        self.device, self.buf = device, {}

    def get(self, name: str, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 16)
        t = self.buf.get(name)
        if t is None or t.numel() < nbytes:
            t = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self.buf[name] = t
        return t


class Signals:
    """The signal matrix resident on one device: rows (m, p), float32 or float64.

    The reference's column-major p x m float64 matrix is row-major (m, p) here.
    float32 storage is used whenever it is exact (every value float32-representable),
    which is the benchmark's case; otherwise float64 keeps arbitrary inputs exact."""

    def __init__(self, rows: torch.Tensor):
        assert rows.dim() == 2 and rows.is_cuda and rows.is_contiguous()
        assert rows.dtype in (torch.float32, torch.float64)
        self.y = rows
        self.m, self.p = rows.shape
        self.code = L.F32 if rows.dtype == torch.float32 else L.F64

    @classmethod
    def from_reference(cls, y: np.ndarray, device, offset: int = 0, count: int | None = None):
        """Upload columns [offset, offset+count) of a p x m float64 matrix."""
        p, m = y.shape
        count = m - offset if count is None else count
        block = y[:, offset:offset + count]
        y32 = block.astype(np.float32)
        exact = np.array_equal(y32.astype(np.float64), block)
        host = np.ascontiguousarray((y32 if exact else block).T)
        return cls(torch.from_numpy(host).to(device))

    @classmethod
    def from_rows(cls, rows: np.ndarray, device):
        return cls(torch.from_numpy(np.ascontiguousarray(rows)).to(device))


@dataclass
class Groups:
    perm: torch.Tensor       # int32 (m,)
    bounds: torch.Tensor     # int64 (K+1,)
    seg_block: torch.Tensor  # int32 (max_seg,)
    seg_lo: torch.Tensor     # int64
    seg_hi: torch.Tensor     # int64
    nseg: torch.Tensor       # int32 (1,)
    max_seg: int
    count: torch.Tensor | None = None  # int64 (1,): positions covered (list tables)

    @property
    def counts(self):
        return self.bounds[1:] - self.bounds[:-1]


@dataclass
class State:
    """Per-signal assignment state after a representation pass."""
    best: torch.Tensor      # int32 (m,)
    score: torch.Tensor     # float64 (m,) energy-pass score of the winner
    norm: torch.Tensor      # float64 (m,) ||y||^2
    residual: torch.Tensor  # float64 (m,) ||y - Q_best x||^2
    total: torch.Tensor     # float64 (1,) local sum of residuals


@dataclass
class IterationOut:
    K: int
    rmse: float
    empty_blocks: list = field(default_factory=list)
    worst: torch.Tensor | None = None


class Engine:
    """One process's device state for a (possibly sharded) SBO problem."""

    def __init__(self, sig: Signals, s0: int, kind: str = "squared-sum", k_cap: int = 64,
                 comm: Comm | None = None, m_total: int | None = None,
                 tc: bool | None = None):
        self.sig, self.s0 = sig, int(s0)
        self.kind = L.KIND[kind]
        self.kind_name = kind
        self.p, self.m = sig.p, sig.m
        self.k = min(self.s0, self.p)
        self.dev = sig.y.device
        self.comm = comm or Comm()
        self.m_total = self.m if m_total is None else int(m_total)
        self.k_cap = int(k_cap)
        self.blocks = torch.zeros((self.k_cap, self.p, self.p), dtype=torch.float64, device=self.dev)
        # right singular vectors of each block's last Procrustes matrix (warm start)
        self.V = torch.empty_like(self.blocks)
        self.K = 0
        self.scratch = Scratch(self.dev)
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.state = State(torch.zeros(self.m, dtype=torch.int32, device=self.dev),
                           torch.zeros(self.m, **f64), torch.zeros(self.m, **f64),
                           torch.zeros(self.m, **f64), torch.zeros(1, **f64))
        self.launches = 0
        self.flag_counts = []
        # state.score holds exact float64 scores for every signal (set by a full
        # representation's residual pass); the incremental re-decision needs them
        self.exact_scores = False
        # tensor-core representation (p = 64): split-fp16 operands, built once
        # tensor-core representation pass: p = 64 (tc_energy.cu) and p = 256 with
        # s0 <= 32 (tc_energy256.cu); other shapes run the float64 tile kernels
        self.i8 = None  # (sy, sx) digit scales of the tensor-core outer product
        self.ci8 = False  # p = 256: the rounds' projection from integer digits
        self.ysy = None   # digit scale of self.ydig (y = Y_int 2^-ysy)
        self.tc = ((self.p == 64 or (self.p == 256 and min(s0, self.p) <= 32))
                   and os.environ.get("SBO_TC", "1") != "0" and self.m > 0
                   and tc is not False)
        if self.tc:
            mp = L.size("sbo_tc_padded_rows", self.m)
            self.yh = torch.zeros((mp, self.p), dtype=torch.float16, device=self.dev)
            self.yl = torch.zeros((mp, self.p), dtype=torch.float16, device=self.dev)
            self.escale = torch.zeros(mp, dtype=torch.int16, device=self.dev)
            self.flags = torch.empty(self.m, dtype=torch.int32, device=self.dev)
            self.nflag = torch.zeros(1, dtype=torch.int32, device=self.dev)
            self._alloc_tc_blocks(self.k_cap)
        self.refresh_signals()

    def refresh_signals(self, rescan: bool = True):
        """Re-derive every device operand of the signals after they changed: the
        tensor-core split (fp16 hi/lo) and the integer digits of the training
        rounds.  ``rescan`` also re-checks the digit format (a host
        synchronisation); pass False when the new signals are known to share the
        old ones' format (e.g. inside a captured CUDA graph): the digit rows are
        then rebuilt in the existing format."""
        if self.tc:
            self._call("sbo_tc_split_signals", self.sig.y.data_ptr(), self.sig.code, self.m,
                       self.p, self.yh.data_ptr(), self.yl.data_ptr(), self.escale.data_ptr(),
                       self.stream)
        if rescan:
            self._scan_digits()
        elif self.ysy is not None:
            self._call("sbo_y_digits", self.sig.y.data_ptr(), self.sig.code, self.m, self.p,
                       self.ysy, self.ydig.data_ptr(), self.stream)

    def _scan_digits(self):
        """Digit formats of the tensor-core outer product (outer_i8.cu): p = 64,
        float32 signals whose values all sit exactly on one fixed-point grid of 35
        bits (unit-range image patches do); otherwise the rounds run the fused
        float64 DMMA kernel."""
        self.i8 = None
        self.ri8 = False
        self.ci8 = False
        self.ysy = None
        if (self.p not in (64, 256) or self.sig.code != L.F32 or self.m == 0
                or os.environ.get("SBO_I8", "1") != "1"):
            return
        out = torch.empty(4, dtype=torch.int32, device=self.dev)
        self._call("sbo_i8_scan", self.sig.y.data_ptr(), self.sig.code, self.m, self.p,
                   out.data_ptr(), self.stream)
        emax, lsb = (int(v) for v in out[:2].cpu())
        norm2 = float(out[2:].view(torch.float64).item())
        if emax < -900:  # every signal is zero
            return
        sy = 35 - emax
        if lsb + sy < 0 or sy > 126 + 35:
            return  # some value is finer than the 35-bit grid: not exact
        self.ysy = sy
        xmax = math.sqrt(norm2) * (1.0 + 1e-6)  # |x| <= ||y|| (orthonormal blocks)
        ex = math.floor(math.log2(xmax)) + 1 if xmax > 0 else 0
        if self.p == 256:
            # p = 256: the rounds' projection from the digits (coef_i8.cu) and the
            # outer product on the 16 (64-dim, 64-atom) slices (outer_i8.cu)
            self.ci8 = os.environ.get("SBO_CI8", "1") == "1"
            if self.ci8:
                if self.k <= 32 and os.environ.get("SBO_OI8_256", "1") == "1":
                    self.i8 = (sy, 54 - ex)
                self.ydig = torch.empty((self.m, 5 * 256), dtype=torch.int8, device=self.dev)
                self._call("sbo_y_digits", self.sig.y.data_ptr(), self.sig.code, self.m,
                           self.p, sy, self.ydig.data_ptr(), self.stream)
            else:
                self.ysy = None
            return
        self.i8 = (sy, 54 - ex)
        # the round's projection from the same digits (k <= 32 selection networks)
        self.ri8 = self.k <= 32 and os.environ.get("SBO_RI8", "1") == "1"
        # signal-major digit rows (5 planes x 64 dims per signal), built once
        self.ydig = torch.empty((self.m, 5 * 64), dtype=torch.int8, device=self.dev)
        self._call("sbo_y_digits", self.sig.y.data_ptr(), self.sig.code, self.m, self.p, sy,
                   self.ydig.data_ptr(), self.stream)

    def _alloc_tc_blocks(self, cap: int):
        self.qh = torch.zeros((cap, self.p, self.p), dtype=torch.float16, device=self.dev)
        self.ql = torch.zeros((cap, self.p, self.p), dtype=torch.float16, device=self.dev)
        self.fscale = torch.zeros(cap, dtype=torch.int16, device=self.dev)

    # ------------------------------------------------------------------ utils
    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.dev).cuda_stream

    def _call(self, name, *args, units: int = 0):
        """One ABI call.  With ``self.timer`` set (bench.py), the call is bracketed
        by CUDA events on this stream and credited with ``units`` signals."""
        self.launches += 1
        t = getattr(self, "timer", None)
        if t is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        L.call(name, *args)
        if t is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            t.append((name, units, e0, e1))
        if L.debug_sync():
            torch.cuda.synchronize(self.dev)

    def set_blocks(self, blocks: np.ndarray | torch.Tensor):
        t = torch.as_tensor(np.asarray(blocks) if not torch.is_tensor(blocks) else blocks,
                            dtype=torch.float64)
        K = t.shape[0]
        self.K = 0
        self.exact_scores = False
        self.ensure_capacity(K)
        self.blocks[:K].copy_(t.to(self.dev))
        self.reset_rotation(0, K)
        self.K = K

    def snapshot(self) -> dict:
        """Device copy of the iteration-entering state (blocks, assignment)."""
        st = self.state
        return {"K": self.K, "blocks": self.blocks.clone(), "exact_scores": self.exact_scores,
                "state": [t.clone() for t in (st.best, st.score, st.norm, st.residual, st.total)]}

    def restore(self, snap: dict):
        """Return to a snapshot's state (device-to-device copies, stream-ordered)."""
        st = self.state
        self.blocks.copy_(snap["blocks"])
        for dst, src in zip((st.best, st.score, st.norm, st.residual, st.total), snap["state"]):
            dst.copy_(src)
        self.K = snap["K"]
        self.exact_scores = snap["exact_scores"]

    def reset_rotation(self, b0: int, b1: int):
        """Identity warm start for the polar Jacobi of blocks [b0, b1)."""
        self.V[b0:b1].copy_(torch.eye(self.p, dtype=torch.float64, device=self.dev).expand(
            b1 - b0, self.p, self.p))

    def v_ptr(self, b: int) -> int:
        return self.V.data_ptr() + b * self.p * self.p * 8

    def ensure_capacity(self, K: int):
        if K > self.V.shape[0]:
            V = torch.empty((K, self.p, self.p), dtype=torch.float64, device=self.dev)
            V[: self.V.shape[0]].copy_(self.V)
            self.V = V
            self.reset_rotation(self.K, K)
        if K > self.k_cap:
            grown = torch.zeros((K, self.p, self.p), dtype=torch.float64, device=self.dev)
            grown[: self.K].copy_(self.blocks[: self.K])
            self.blocks, self.k_cap = grown, K

    def block_ptr(self, b: int) -> int:
        return self.blocks.data_ptr() + b * self.p * self.p * 8

    # ------------------------------------------------------ representation
    def energy(self, b0: int, b1: int, accumulate: bool):
        s = self.state
        if self.tc:
            # tensor-core pass over [b0, b1), then exact float64 re-decision of
            # the signals whose certificate failed (near-ties)
            if self.qh.shape[0] < self.k_cap:
                self._alloc_tc_blocks(self.k_cap)
            # operands of the blocks this pass reads, [b0, b1)
            pp = self.p * self.p
            self._call("sbo_tc_split_blocks", self.blocks.data_ptr() + 8 * b0 * pp, b1 - b0,
                       self.p, self.qh.data_ptr() + 2 * b0 * pp,
                       self.ql.data_ptr() + 2 * b0 * pp, self.fscale.data_ptr() + 2 * b0,
                       self.stream)
            self.nflag.zero_()
            # <= 64 blocks: the flagged signals carry candidate-block masks (full
            # pass: the blocks within the certificate's tolerance of the best;
            # incremental pass: the incoming winner and the appended blocks);
            # sorted by them, the float64 tiles only visit their union.  Every
            # candidate is re-evaluated by the same float64 kernel, so exact ties
            # go to the lower block (sbo.py:191) whatever kernel produced the
            # stored scores.
            use_cand = b1 <= 64
            if use_cand and getattr(self, "cand", None) is None:
                i32 = dict(dtype=torch.int32, device=self.dev)
                i64 = dict(dtype=torch.int64, device=self.dev)
                self.cand = torch.empty(self.m, **i64)          # 64-bit block masks
                self.flags_sorted = torch.empty(self.m, **i32)
                self.cand_sorted = torch.empty(self.m, **i64)
            self._call("sbo_tc_energy" if self.p == 64 else "sbo_tc_energy256",
                       self.yh.data_ptr(), self.yl.data_ptr(),
                       self.escale.data_ptr(), self.m, self.qh.data_ptr(), self.ql.data_ptr(),
                       self.fscale.data_ptr(), b0, b1, self.s0, self.kind, int(accumulate),
                       s.best.data_ptr(), s.score.data_ptr(), s.residual.data_ptr(),
                       self.flags.data_ptr(), self.nflag.data_ptr(),
                       self.cand.data_ptr() if use_cand else None, self.stream,
                       units=self.m * (b1 - b0))
            if use_cand:
                ws = self.scratch.get("cand", L.size("sbo_cand_workspace_bytes"))
                self._call("sbo_cand_sort", self.flags.data_ptr(), self.cand.data_ptr(),
                           self.nflag.data_ptr(), self.m, self.flags_sorted.data_ptr(),
                           self.cand_sorted.data_ptr(), ws.data_ptr(), ws.numel(), self.stream)
                if (self.ci8 and not accumulate
                        and os.environ.get("SBO_RECHECK_PAIRS", "1") == "1"):
                    # p = 256, full pass: per-(signal, candidate block) pairs,
                    # projected from the integer digits block by block (the
                    # incremental pass's masks are the incoming winner and the
                    # appended block: its tile unions are already tight)
                    ws = self.scratch.get("rpairs", L.size("sbo_recheck_pairs_workspace_bytes",
                                                           b1, self.m))
                    self._call("sbo_energy_recheck_pairs", self.ydig.data_ptr(), self.ysy,
                               self.blocks.data_ptr(), b1, self.s0, self.kind,
                               self.flags_sorted.data_ptr(), self.cand_sorted.data_ptr(),
                               self.nflag.data_ptr(), self.m, s.best.data_ptr(),
                               s.score.data_ptr(), s.residual.data_ptr(), ws.data_ptr(),
                               ws.numel(), self.stream)
                elif self.ci8:  # p = 256: tiles over the union of their masks
                    ws = self.scratch.get("rci8", L.size("sbo_recheck_i8_workspace_bytes", b1))
                    self._call("sbo_energy_recheck_i8", self.ydig.data_ptr(), self.ysy,
                               self.blocks.data_ptr(), b1, self.s0, self.kind,
                               self.flags_sorted.data_ptr(), self.cand_sorted.data_ptr(),
                               self.nflag.data_ptr(), self.m, s.best.data_ptr(),
                               s.score.data_ptr(), s.residual.data_ptr(), ws.data_ptr(),
                               ws.numel(), self.stream)
                else:
                    self._call("sbo_energy_recheck_cand", self.sig.y.data_ptr(),
                               self.sig.code, self.m, self.p, self.blocks.data_ptr(), b1,
                               self.s0, self.kind, self.flags_sorted.data_ptr(),
                               self.cand_sorted.data_ptr(), self.nflag.data_ptr(), self.m,
                               s.best.data_ptr(), s.score.data_ptr(), s.residual.data_ptr(),
                               self.stream)
            else:
                # more than 64 blocks: the flagged signals are re-decided over every
                # block from scratch
                self._call("sbo_energy_recheck", self.sig.y.data_ptr(), self.sig.code, self.m,
                           self.p, self.blocks.data_ptr(), 0, b1,
                           self.s0, self.kind, self.flags.data_ptr(), self.nflag.data_ptr(),
                           self.m, s.best.data_ptr(), s.score.data_ptr(),
                           s.residual.data_ptr(), self.stream)
            self.flag_counts = self.flag_counts[-7:] + [self.nflag.clone()]
            self.exact_scores = False
            return
        self._call("sbo_energy_pass", self.sig.y.data_ptr(), self.sig.code, self.m, self.p,
                   self.blocks.data_ptr(), b0, b1, self.s0, self.kind, int(accumulate),
                   s.best.data_ptr(), s.score.data_ptr(), s.residual.data_ptr(),
                   None if accumulate else s.norm.data_ptr(), self.stream)

    def residual(self):
        """Deterministic sum of the squared residuals (the RMSE numerator)."""
        s = self.state
        ws = self.scratch.get("sum", L.size("sbo_sum_workspace_bytes", self.m))
        self._call("sbo_sum", s.residual.data_ptr(), self.m, s.total.data_ptr(), ws.data_ptr(),
                   ws.numel(), self.stream)

    def group(self, K: int) -> Groups:
        sl = seg_len(self.m)
        max_seg = L.size("sbo_max_segments", self.m, K, sl)
        d = self.dev
        g = Groups(torch.empty(max(self.m, 1), dtype=torch.int32, device=d),
                   torch.empty(K + 1, dtype=torch.int64, device=d),
                   torch.empty(max_seg, dtype=torch.int32, device=d),
                   torch.empty(max_seg, dtype=torch.int64, device=d),
                   torch.empty(max_seg, dtype=torch.int64, device=d),
                   torch.zeros(1, dtype=torch.int32, device=d), max_seg)
        ws = self.scratch.get("group", L.size("sbo_group_workspace_bytes", self.m, K))
        self._call("sbo_group", self.state.best.data_ptr(), self.m, K, sl,
                   g.perm.data_ptr(), g.bounds.data_ptr(), g.seg_block.data_ptr(),
                   g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(), ws.data_ptr(),
                   ws.numel(), self.stream)
        return g

    def list_segments(self, n: int, count: torch.Tensor | None = None) -> Groups:
        """Segment table of a single list of n entries (a member list); with
        ``count`` (int64 device tensor), of its first min(n, count) entries,
        built on the device (no host read of the count)."""
        sl = seg_len(n)
        if count is not None:
            max_seg = max(1, math.ceil(n / sl))
            g = Groups(None, None, torch.zeros(max_seg, dtype=torch.int32, device=self.dev),
                       torch.empty(max_seg, dtype=torch.int64, device=self.dev),
                       torch.empty(max_seg, dtype=torch.int64, device=self.dev),
                       torch.zeros(1, dtype=torch.int32, device=self.dev), max_seg)
            self._call("sbo_chunk_segments", n, count.data_ptr(), sl, g.seg_lo.data_ptr(),
                       g.seg_hi.data_ptr(), g.nseg.data_ptr(), self.stream)
            g.count = count
            return g
        nseg = max(1, math.ceil(n / sl)) if n > 0 else 0
        lo = torch.arange(0, max(n, 1), sl, dtype=torch.int64, device=self.dev)[:nseg]
        hi = torch.clamp(lo + sl, max=n)
        # torch.full, not torch.tensor: no pageable host->device copy (which would
        # synchronise the host with the queued kernels mid-iteration)
        return Groups(None, None, torch.zeros(max(nseg, 1), dtype=torch.int32, device=self.dev),
                      lo, hi, torch.full((1,), nseg, dtype=torch.int32, device=self.dev),
                      max(nseg, 1))

    def code(self, order, g: Groups, block_override: int, out_by_signal: bool, ld: int,
             idx, val, energy=None, kept=None):
        self._call("sbo_code_segments", self.sig.y.data_ptr(), self.sig.code, self.p,
                   _ptr(order), g.seg_block.data_ptr(), g.seg_lo.data_ptr(),
                   g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg, self.blocks.data_ptr(),
                   block_override, self.s0, self.kind, int(out_by_signal), ld,
                   _ptr(idx), _ptr(val), _ptr(energy), _ptr(kept), self.stream,
                   units=self.m if order is not None and g.bounds is not None else 0)

    def code_i8(self, order, g: Groups, n: int, nblocks: int, block_override: int, ld: int,
                idx, val, energy=None, kept=None, by_signal: bool = False, count=None):
        """``code`` for p = 256 with the projection on the tensor cores: exact
        integer-digit coefficients of every position (coef_i8.cu), then the
        float64 selection of sbo_code_segments on them (sbo_select_coded)."""
        nb = block_override + 1 if block_override >= 0 else nblocks
        ws = self.scratch.get("ci8", L.size("sbo_coef_i8_workspace_bytes", nb))
        coef = self.scratch.get("coef", 8 * max(n, 1) * self.p)
        self._call("sbo_coef_i8_segments", self.ydig.data_ptr(), self.ysy, _ptr(order),
                   g.seg_block.data_ptr(), g.seg_lo.data_ptr(), g.seg_hi.data_ptr(),
                   g.nseg.data_ptr(), g.max_seg, self.blocks.data_ptr(), nb, block_override,
                   coef.data_ptr(), ws.data_ptr(), ws.numel(), self.stream, units=n)
        self._call("sbo_select_coded", coef.data_ptr(), _ptr(count), n, self.p, self.s0,
                   self.kind, _ptr(order) if by_signal else None, ld, _ptr(idx), _ptr(val),
                   _ptr(energy), _ptr(kept), self.stream, units=n)

    # ----------------------------------------------------------- training
    def train_rounds(self, order, g: Groups, n: int, rounds: int, nblocks: int,
                     first_block: int, counts, status: torch.Tensor, single: bool):
        """R rounds of (code, P = Y X^T, allreduce, polar) for `nblocks` blocks.

        single=True: one block (first_block) over a member list of n entries."""
        p = self.p
        partial = (self.scratch.get("partial", 8 * g.max_seg * p * p) if self.i8 is None
                   else None)
        i8_ws = ytiles = None
        if self.i8 is not None:
            i8_ws = self.scratch.get("i8", L.size("sbo_outer_i8_workspace_bytes", nblocks, p))
            # transposed digit tiles of this grouping, shared by its R rounds
            ytiles = self.scratch.get("ytiles_list" if single else "ytiles",
                                      L.size("sbo_y_tiles_bytes", n, g.max_seg, p))
            self._call("sbo_y_tiles", self.ydig.data_ptr(), p, _ptr(order), g.seg_lo.data_ptr(),
                       g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg, ytiles.data_ptr(),
                       self.stream, units=n)
        P = self.scratch.get("P", 8 * nblocks * p * p)
        ld = max(n, 1)
        idx = self.scratch.get("tr_idx", 2 * self.k * ld).view(torch.int16)
        val = self.scratch.get("tr_val", 8 * self.k * ld).view(torch.float64)
        pol_ws = self.scratch.get("polar", L.size("sbo_polar_workspace_bytes", nblocks, p))
        Pt = P[: 8 * nblocks * p * p].view(torch.float64).view(nblocks, p, p)
        fused = p <= 64 and os.environ.get("SBO_FUSED_ROUND", "1") != "0"
        override = first_block if single else -1
        for r in range(rounds):
            if self.i8 is not None:
                # coding (float64 DMMA projection, exact selection) writes the kept
                # pairs; P = Y X^T on tcgen05 from exact integer digits
                if self.ri8:
                    # the projection on tcgen05 from exact integer digits
                    nb = first_block + 1 if single else nblocks
                    ws = self.scratch.get("ri8", L.size("sbo_round_i8_workspace_bytes", nb))
                    self._call("sbo_round_i8_segments", self.ydig.data_ptr(), self.i8[0],
                               _ptr(order), g.seg_block.data_ptr(), g.seg_lo.data_ptr(),
                               g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg,
                               self.blocks.data_ptr(), nb, override, self.s0, 0, self.kind,
                               ld, idx.data_ptr(), val.data_ptr(), None, None, ws.data_ptr(),
                               ws.numel(), self.stream, units=n)
                elif self.ci8:  # p = 256
                    self.code_i8(order, g, n, nblocks, first_block if single else -1, ld,
                                 idx, val, count=g.count)
                else:
                    self._call("sbo_round_code_segments", self.sig.y.data_ptr(),
                               self.sig.code, p, _ptr(order), g.seg_block.data_ptr(),
                               g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(),
                               g.max_seg, self.blocks.data_ptr(), override, self.s0, ld,
                               idx.data_ptr(), val.data_ptr(), self.stream, units=n)
                self._call("sbo_outer_i8_segments", ytiles.data_ptr(), p,
                           None if single else g.seg_block.data_ptr(), g.seg_lo.data_ptr(),
                           g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg, nblocks,
                           self.s0, ld, idx.data_ptr(), val.data_ptr(), self.i8[0],
                           self.i8[1], Pt.data_ptr(), i8_ws.data_ptr(), i8_ws.numel(),
                           self.stream, units=n)
            elif fused:  # coding + P partials in one pass per segment
                self._call("sbo_round_segments", self.sig.y.data_ptr(), self.sig.code, p,
                           _ptr(order), g.seg_block.data_ptr(), g.seg_lo.data_ptr(),
                           g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg,
                           self.blocks.data_ptr(), override, self.s0, partial.data_ptr(),
                           self.stream, units=n)
            else:
                if self.ci8:
                    self.code_i8(order, g, n, nblocks, first_block if single else -1, ld,
                                 idx, val, count=g.count)
                else:
                    self.code(order, g, override, False, ld, idx, val)
                self._call("sbo_outer_segments", self.sig.y.data_ptr(), self.sig.code, p,
                           _ptr(order), g.seg_lo.data_ptr(), g.seg_hi.data_ptr(),
                           g.nseg.data_ptr(), g.max_seg, self.s0, ld, idx.data_ptr(),
                           val.data_ptr(), partial.data_ptr(), self.stream, units=n)
            if self.i8 is None:
                self._call("sbo_reduce_segments", partial.data_ptr(),
                           None if single else g.seg_block.data_ptr(), g.nseg.data_ptr(),
                           g.max_seg, nblocks, p, Pt.data_ptr(), self.stream)
            self.comm.allreduce(Pt)
            self._call("sbo_polar", Pt.data_ptr(), nblocks, p, _ptr(counts),
                       self.block_ptr(first_block), self.v_ptr(first_block), None,
                       status[r].data_ptr(), pol_ws.data_ptr(), pol_ws.numel(), self.stream,
                       units=nblocks)

    def gram(self, members, w: int, count: torch.Tensor | None = None) -> torch.Tensor:
        G = torch.empty((self.p, self.p), dtype=torch.float64, device=self.dev)
        chunk = seg_len(w)
        ws = self.scratch.get("gram", L.size("sbo_gram_workspace_bytes", w, chunk, self.p))
        self._call("sbo_gram_counted", self.sig.y.data_ptr(), self.sig.code, self.p,
                   _ptr(members), w, _ptr(count), chunk, G.data_ptr(), ws.data_ptr(),
                   ws.numel(), self.stream)
        return G

    def init_block(self, G, ncols: int, draws: np.ndarray, slot: int, status, rank=None):
        self.reset_rotation(slot, slot + 1)
        if torch.is_tensor(draws) and draws.is_cuda:  # already staged on the device
            d = draws.to(torch.float64).contiguous()
            ws = self.scratch.get("init", L.size("sbo_init_workspace_bytes", self.p))
            self._call("sbo_init_block", G.data_ptr(), self.p, ncols, d.data_ptr(), d.shape[0],
                       self.block_ptr(slot), _ptr(rank), status.data_ptr(), ws.data_ptr(),
                       ws.numel(), self.stream)
            return
        # staged through a persistent pinned buffer and copied asynchronously (a
        # pageable copy would synchronise); the buffer is reused only after the
        # iteration's closing synchronisation
        host = np.ascontiguousarray(draws, dtype=np.float64)
        pin = getattr(self, "_draws_pin", None)
        done = getattr(self, "_draws_done", None)
        if done is not None:
            done.synchronize()  # the previous copy out of the buffer has run
        if pin is None or pin.numel() < host.size:
            pin = self._draws_pin = torch.empty(host.size, dtype=torch.float64).pin_memory()
        pin[: host.size].copy_(torch.from_numpy(host.reshape(-1)))
        d = torch.empty(host.shape, dtype=torch.float64, device=self.dev)
        d.view(-1).copy_(pin[: host.size], non_blocking=True)
        self._draws_done = torch.cuda.Event()
        self._draws_done.record()
        ws = self.scratch.get("init", L.size("sbo_init_workspace_bytes", self.p))
        self._call("sbo_init_block", G.data_ptr(), self.p, ncols, d.data_ptr(), d.shape[0],
                   self.block_ptr(slot), _ptr(rank), status.data_ptr(), ws.data_ptr(),
                   ws.numel(), self.stream)

    def worst(self, w: int) -> tuple[torch.Tensor, int, torch.Tensor | None]:
        """Local members of the global worst-w set (ascending signal order):
        (members, n, count).  One GPU: n members.  Sharded: at most n members,
        the local count in the device tensor ``count`` (never read back here)."""
        res = self.state.residual
        if self.comm.world == 1 and not getattr(self.comm, "sharded", False):
            n = min(w, self.m)
            members = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
            ws = self.scratch.get("worst", L.size("sbo_worst_workspace_bytes", self.m))
            self._call("sbo_worst_set", res.data_ptr(), self.m, w, members.data_ptr(),
                       ws.data_ptr(), ws.numel(), self.stream)
            return members, n, None
        return distributed_worst(self, w)

    # ----------------------------------------------------------- iteration
    def represent_full(self):
        """Full representation: winners, then exact float64 squared residuals."""
        self.energy(0, self.K, False)
        if self.tc:
            # the tensor-core pass certifies the winner; its residual is only
            # float32-accurate, so recode every signal in its winning block in
            # float64 (exact support + discarded energy), as the worst set needs
            g = self.group(self.K)
            if self.ri8:
                ws = self.scratch.get("ri8", L.size("sbo_round_i8_workspace_bytes", self.K))
                self._call("sbo_round_i8_segments", self.ydig.data_ptr(), self.i8[0],
                           g.perm.data_ptr(), g.seg_block.data_ptr(), g.seg_lo.data_ptr(),
                           g.seg_hi.data_ptr(), g.nseg.data_ptr(), g.max_seg,
                           self.blocks.data_ptr(), self.K, -1, self.s0, 1, self.kind, 0,
                           None, None, self.state.residual.data_ptr(),
                           self.state.score.data_ptr(), ws.data_ptr(), ws.numel(),
                           self.stream, units=self.m)
            elif self.p <= 64:
                self._call("sbo_residual_segments", self.sig.y.data_ptr(), self.sig.code,
                           self.p, g.perm.data_ptr(), g.seg_block.data_ptr(),
                           g.seg_lo.data_ptr(), g.seg_hi.data_ptr(), g.nseg.data_ptr(),
                           g.max_seg, self.blocks.data_ptr(), self.s0, self.kind,
                           self.state.residual.data_ptr(), self.state.score.data_ptr(),
                           self.stream, units=self.m)
            elif self.ci8:
                self.code_i8(g.perm, g, self.m, self.K, -1, max(self.m, 1), None, None,
                             self.state.score, self.state.residual, by_signal=True)
            else:
                ld = max(self.m, 1)
                self.code(g.perm, g, -1, True, ld, None, None, self.state.score,
                          self.state.residual)
        self.exact_scores = True
        self.residual()

    def rmse(self) -> float:
        tot = self.comm.allreduce(self.state.total.clone())
        return math.sqrt(max(float(tot.item()), 0.0) / (self.p * self.m_total))

    def iterate(self, w: int, rounds: int, draws, timer=None,
                force_new_block: np.ndarray | None = None) -> IterationOut:
        """One SBO iteration (sbo.py:352-397) entering with self.K blocks.

        ``timer.mark()`` (optional) is called at the phase boundaries: start, new
        block trained, represent #1, retrain, represent #2.  ``force_new_block``
        (tests only) replaces the trained new block — teacher forcing past a
        rank-deficient Procrustes step, whose polar factor is not unique."""
        dev_out = self.iterate_device(w, rounds, draws, timer, force_new_block)
        return self.finish_iteration(dev_out)

    def iterate_device(self, w: int, rounds: int, draws, timer=None,
                       force_new_block: np.ndarray | None = None) -> dict:
        """The device work of one iteration, with no host synchronisation (CUDA-graph
        capturable on one GPU when ``draws`` is already a device tensor)."""
        mark = timer.mark if timer is not None else (lambda: None)
        mark()
        K0 = self.K
        self.ensure_capacity(K0 + 1)
        self.reset_rotation(K0, K0 + 1)
        st = torch.zeros((2, rounds + 1, K0 + 1), dtype=torch.int32, device=self.dev)
        # worst set and the new block (sbo.py:353-357)
        members, n, count = self.worst(w)
        if force_new_block is None:
            n_total = min(w, self.m_total)
            G = self.comm.allreduce(self.gram(members, n, count))
            self.init_block(G, n_total, draws, K0, st[0, rounds, :1])
            segs = self.list_segments(n, count)
            self.train_rounds(members, segs, n, rounds, 1, K0, None, st[0], single=True)
        else:
            self.blocks[K0].copy_(torch.as_tensor(force_new_block, dtype=torch.float64))
        self.K = K0 + 1
        mark()
        # represent #1: only the appended block can change a winner (sbo.py:361)
        self.energy(K0, K0 + 1, True)
        mark()
        # group + retrain every block on its signals (sbo.py:367-385)
        g = self.group(self.K)
        counts = g.counts
        if self.comm.world > 1:
            counts = self.comm.allreduce(counts.clone())
        self.train_rounds(g.perm, g, self.m, rounds, self.K, 0, counts, st[1], single=False)
        mark()
        # represent #2 (sbo.py:389-394)
        self.represent_full()
        mark()
        return {"status": st, "counts": counts, "members": members, "n": n, "count": count,
                "K": self.K}

    def finish_iteration(self, d: dict) -> IterationOut:
        """Host side of an iteration: RMSE, status checks, empty-block list."""
        self.K = d["K"]
        rmse = self.rmse()
        stc = d["status"].cpu().numpy()
        cnt = d["counts"].cpu().numpy()
        # Jacobi sweeps / Newton-Schulz iterations per (phase, round, block)
        self.last_sweeps = (stc >> 8) & 0xFF
        check_status(stc, self.p)
        empty = [b for b in range(self.K) if cnt[b] == 0]
        n = d["n"] if d.get("count") is None else int(d["count"].item())
        return IterationOut(self.K, rmse, empty, d["members"][:n])

    def capture(self, fn, prepare):
        """CUDA graph of ``fn()`` (device work only) after two eager warm-up runs on a
        side stream, each preceded by ``prepare()``; ``prepare()`` also runs once
        before the capture.  Returns (graph, the value fn returned while captured)."""
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            for _ in range(2):
                prepare()
                fn()
        torch.cuda.current_stream(self.dev).wait_stream(side)
        torch.cuda.synchronize(self.dev)
        prepare()
        torch.cuda.synchronize(self.dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            out = fn()
        torch.cuda.synchronize(self.dev)
        return graph, out

    def capture_iteration(self, snapshot: dict, w: int, rounds: int, draws_dev: torch.Tensor):
        """CUDA graph of (restore the snapshot; one iteration's device work) for
        repeated iterations from the same entering state on one GPU (the bench):
        replaying it removes the host launch gaps between the ~100 kernels.
        Returns replay() -> IterationOut."""
        if ((self.comm.world > 1 or getattr(self.comm, "sharded", False))
                and not getattr(self.comm, "capturable", False)):
            raise ValueError("graph capture of a sharded iteration needs NCCL collectives "
                             "(gloo exchanges go through the host)")
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):  # warm-up: scratch sizes, kernel attributes
            for _ in range(2):
                self.restore(snapshot)
                self.iterate_device(w, rounds, draws_dev)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        torch.cuda.synchronize(self.dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.restore(snapshot)
            out = self.iterate_device(w, rounds, draws_dev)
        torch.cuda.synchronize(self.dev)

        def replay() -> IterationOut:
            graph.replay()
            return self.finish_iteration(out)

        replay.graph = graph
        return replay


def check_status(st: np.ndarray, p: int | None = None):
    """Map the device status words of the polar / init steps onto the reference's
    exceptions (linalg.py:61-63 names the matrix dimensions; onb.py:119-124)."""
    from .linalg import DecompositionError
    from .onb import NumericalError
    st = np.asarray(st) & 0xFF  # bits 8.. carry the Jacobi sweep count
    if (st == L.ST_NOCONV).any():
        dims = f"a {p}x{p} matrix" if p else "a block update"
        raise DecompositionError(f"SVD did not converge for {dims}")
    if (st == L.ST_DEFECT).any():
        raise NumericalError("block lost orthonormality: defect > 1e-08")


def distributed_worst(eng: Engine, w: int) -> tuple[torch.Tensor, int, torch.Tensor]:
    """Global worst-w across ranks: radix select with allreduced 256-bin histograms.

    Keys are the float64 bit patterns of residual_sq (order-preserving for >= 0);
    ties at the threshold go to the lowest GLOBAL signal index, i.e. to lower
    ranks first (contiguous column shards) — dist.equal_quota's rule, applied on
    the device.  The select state, the eight histograms and the tie counts stay in
    device memory (collectives stream-ordered on NCCL), and so does the local
    member count: the Gram and the segment table read it on the device, launches
    are sized by the bound min(w, m_local) — no host synchronisation, so the
    sharded iteration can be captured as a CUDA graph on NCCL."""
    res = eng.state.residual
    need = min(w, eng.m_total)
    members = torch.empty(max(eng.m, 1), dtype=torch.int32, device=eng.dev)
    count = torch.zeros(1, dtype=torch.int64, device=eng.dev)
    if need < 1:
        return members, 0, count
    ws = eng.scratch.get("worst", L.size("sbo_worst_workspace_bytes", eng.m))
    hist = torch.empty(256, dtype=torch.int64, device=eng.dev)
    eng._call("sbo_select_begin", ws.data_ptr(), need, eng.stream)
    for shift in range(56, -8, -8):
        eng._call("sbo_select_hist", res.data_ptr(), eng.m, ws.data_ptr(), shift,
                  hist.data_ptr(), eng.stream)
        eng.comm.allreduce(hist)
        eng._call("sbo_select_pick", ws.data_ptr(), hist.data_ptr(), shift, eng.stream)
    gt_eq = torch.empty(2, dtype=torch.int64, device=eng.dev)
    eng._call("sbo_select_counts", res.data_ptr(), eng.m, ws.data_ptr(), ws.numel(),
              gt_eq.data_ptr(), eng.stream)
    eq_all = eng.comm.allgather(gt_eq[1:2].clone())
    eng._call("sbo_select_write", res.data_ptr(), eng.m, ws.data_ptr(), ws.numel(),
              gt_eq.data_ptr(), eq_all.data_ptr(), eng.comm.rank, members.data_ptr(),
              count.data_ptr(), eng.stream)
    return members, min(need, eng.m), count
