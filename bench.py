#!/usr/bin/env python
"""Benchmark: signals/s of one SBO iteration (p=64, K=16, s0=8) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one ``sbo_train`` loop-body iteration (sbo.py:352-397) entering with
K-1 = 15 blocks and leaving with K = 16, over m = 2^24 synthetic 8x8 image
patches of a 4096^2 scene (BASELINE.json config C), sharded by contiguous
columns over the N GPUs (strong scaling: m/N signals per GPU).  Every step
restores the same entering state.  Prints ONE JSON line on rank 0.

``--gpus N`` with N > 1 outside torchrun re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU, NCCL); with
SBO_BENCH_ONE_GPU=1 every rank shares cuda:0 over gloo (a functional check of
the sharded path on a one-GPU box, not a performance configuration).
``--impl reference`` times the reference algorithm on the host cores instead
(the CPU oracle port on a 2^20-signal sample of the workload; rank 0 only).
"""
from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import math  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "signals/sec per SBO iteration (p=64,K=16,s0=8) at 1/2/4/8 B200 vs CPU ref"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    # (not "--m": torch.distributed.run rejects it as an ambiguous prefix when
    # --gpus N re-launches this script)
    ap.add_argument("--m-total", dest="m_total", type=int, default=1 << 24,
                    help="signals in the whole job (config C: 2^24)")
    ap.add_argument("--m-per-gpu", dest="m_per_gpu", type=int, default=None,
                    help="weak scaling: signals per GPU (overrides --m)")
    ap.add_argument("--p-edge", type=int, default=8)
    ap.add_argument("--K", type=int, default=16)
    ap.add_argument("--s0", type=int, default=8)
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--scene", type=int, default=4096)
    ap.add_argument("--cpu-sample", type=int, default=1 << 20)
    ap.add_argument("--cpu-steps", type=int, default=3,
                    help="timed CPU iterations (each one a --cpu-sample iteration)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()
    a.world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.m_per_gpu is not None:
        a.scaling, a.m_total = "weak", a.m_per_gpu * max(a.world, 1)
    else:
        a.scaling = "strong"
    return a


def config_label(a):
    std = {(64, 16, 8, 1 << 24): "C", (64, 16, 8, 1 << 20): "B", (256, 32, 16, 1 << 22): "D"}
    key = (a.p_edge ** 2, a.K, a.s0, a.m_total)
    return std.get(key, "E" if (a.p_edge == 8 and a.m_total == 1 << 22) else "custom")


def workload_name(a, world):
    return (f"{config_label(a)}: p={a.p_edge**2}, K={a.K} (entering {a.K - 1}), s0={a.s0}, "
            f"R={a.rounds}, m=2^{math.log2(a.m_total):g} total over {world} GPU(s) "
            f"({a.scaling} scaling, {a.m_total // world} per GPU), W=m/16, "
            f"{a.p_edge}x{a.p_edge} patches of a {a.scene}^2 synthetic scene")


def shard_range(a, rank, world):
    """Contiguous column shard [lo, hi) of rank (the first m % world ranks get one more)."""
    base, extra = divmod(a.m_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_signals(a, rank, world):
    from paper_1412_4944_b200 import signals
    grid = signals.scene(a.scene, a.scene, 0)
    lo, hi = shard_range(a, rank, world)
    u8 = signals.patch_bytes(grid, a.p_edge, a.m_total, 11, lo, hi)
    return signals.unit_range(u8), a.m_total


def relaunch_args(gpus: int, port: int, argv: list[str]) -> list[str]:
    """torch.distributed.run arguments that re-run this script with `argv` on
    `gpus` ranks (tests/test_bench_cli.py: every bench option survives the
    launcher's own parser)."""
    return ["--nnodes=1", f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1",
            f"--master-port={port}", str(Path(__file__).resolve())] + list(argv)


def relaunch_distributed(a):
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run"] + relaunch_args(a.gpus, port,
                                                                          sys.argv[1:])
    sys.exit(subprocess.call(cmd))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc = index, None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


# Algorithmic work per unit of each timed ABI call:
#   round  (sbo_round_segments, unit = signal):  own-block projection 2p^2 +
#          sparse outer product 2 p k — the reference's train_onb round
#   tc     (sbo_tc_energy, unit = signal x block): projection 2p^2
#   code   (sbo_code_segments, unit = signal): projection 2p^2
FP64_PEAK_TFLOPS = 33.0       # measured DFMA throughput on this pool (profiles/fp64_micro.txt)
DMMA_PEAK_TFLOPS = 37.0       # measured float64 tensor-core (DMMA m8n8k4) throughput, same file
I8_PEAK_TOPS = 4188.7         # measured tcgen05 kind::i8 dense throughput (profiles/i8_micro.txt)


def kernel_families(timer, p, k):
    """Per ABI-call family: launches, time, algorithmic flop rate (the reference's
    work: sparse outer product 2pk) and implemented flop rate (what the kernel
    issues: dense DMMA outer product 2p^2; three fp16 products in the split)."""
    fam = {"sbo_round_segments": ("k_round64", 2 * p * p + 2 * p * k, 4 * p * p,
                                  "fp64 tensor cores (DMMA)"),
           "sbo_tc_energy": ("k_energy_tc", 2 * p * p, 6 * p * p, "tcgen05 split-fp16"),
           "sbo_round_code_segments": ("k_round64<code>", 2 * p * p, 2 * p * p,
                                       "fp64 tensor cores (DMMA)"),
           # 1920 digit-product columns x 64 dims x 2 int8 ops per signal (round_i8.cu)
           "sbo_round_i8_segments": ("k_round_i8", 2 * p * p, 2 * 64 * 1920,
                                     "tcgen05 kind::i8 (exact integer digits)"),
           # 1280 digit-product columns x 128 rows x 2 int8 ops per signal and 64 x 64
           # slice (outer_i8.cu; p = 256: 16 slices)
           "sbo_outer_i8_segments": ("k_outer_i8", 2 * p * k, 2 * 128 * 1280 * (p // 64) ** 2,
                                     "tcgen05 kind::i8 (exact integer digits)"),
           "sbo_code_segments": ("k_code_f64", 2 * p * p, 2 * p * p, "fp64 CUDA cores"),
           "sbo_residual_segments": ("k_round64<resid>", 2 * p * p, 2 * p * p,
                                     "fp64 tensor cores (DMMA)"),
           "sbo_tc_energy256": ("k_energy_tc256", 2 * p * p, 6 * p * p, "tcgen05 split-fp16"),
           # p = 256: 7680 digit-product columns x 256 atoms x 2 int8 ops per signal
           # (coef_i8.cu: 16 stages x 2 k-steps x 1920 columns x 32 deep x 2 / 256)
           "sbo_coef_i8_segments": ("k_coef_i8", 2 * p * p, 2 * 256 * 7680,
                                    "tcgen05 kind::i8 (exact integer digits)"),
           "sbo_select_coded": ("k_select_coded", 0, 0, "fp64 CUDA cores, selection"),
           # p = 256: the kept pairs only (k_outer_sparse256); p <= 64: dense DMMA
           "sbo_outer_segments": ("k_outer_sparse256" if p == 256 else "k_outer_f64",
                                  2 * p * k, 2 * p * k if p == 256 else 2 * p * p,
                                  "fp64 CUDA cores (kept pairs)" if p == 256
                                  else "fp64 tensor cores (DMMA)"),
           "sbo_polar": ("k_polar_ns_cluster", 0, 0, "fp64 tensor cores (DMMA), latency"),
           "sbo_energy_recheck": ("k_energy_f64 recheck", 0, 0, "fp64 tensor cores (DMMA)"),
           "sbo_energy_recheck_cand": ("k_energy_f64 recheck (candidates)", 0, 0,
                                       "fp64 tensor cores (DMMA)")}
    out = {}
    for name, (kname, fpu, ipu, pipe) in fam.items():
        ev = [(u, e0.elapsed_time(e1)) for (n, u, e0, e1) in timer if n == name]
        if not ev:
            continue
        ms = sum(t for _, t in ev)
        units = sum(u for u, _ in ev)
        out[kname] = {"launches": len(ev), "ms_total": ms, "units": units,
                      "flop_per_unit": fpu, "implemented_flop_per_unit": ipu, "pipe": pipe,
                      "tflops": (fpu * units / (ms * 1e-3) / 1e12) if fpu and ms else None,
                      "implemented_tflops": (ipu * units / (ms * 1e-3) / 1e12) if ipu and ms
                      else None}
    return out


def ncu_traffic(kname):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kname` from the
    newest committed ncu --set full summary (profiles/*_ncu_summary.txt), or None."""
    import glob
    files = sorted(glob.glob(str(ROOT / "profiles" / "*_ncu_summary.txt")))
    want = {"k_round64": "k_round64<float, 0>", "k_round64<resid>": "k_round64<float, 1>",
            "k_energy_tc": "k_energy_tc<", "k_round_i8": "k_round_i8<",
            "k_outer_i8": "k_outer_i8"}.get(kname)
    if not files or not want:
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    cur, total, path = None, {}, files[-1]
    for line in open(path):
        if line.startswith("=="):
            cur = want in line
            total = {} if cur else total
            continue
        f = line.split()
        if cur and len(f) >= 3 and f[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total[f[0]] = float(f[1]) * scale.get(f[2], 1.0)
        if cur and len(total) == 2:
            return {"bytes_per_launch": sum(total.values()), "source": os.path.basename(path)}
    return None


def roofline_of(kname, info, bf16, src, steps):
    achieved = info["tflops"] or 0.0
    tr = ncu_traffic(kname)
    return {"kernel": kname, "bound": "tensor", "achieved": achieved, "peak": bf16,
            "unit": "TFLOP/s", "frac": achieved / bf16,
            "traffic": tr["bytes_per_launch"] if tr else None,
            "traffic_source": tr["source"] if tr else None,
            "peak_source": f"{src} bf16 dense (MEASURED_PEAKS.json)",
            "fp64_peak": FP64_PEAK_TFLOPS,
            "frac_of_fp64_peak": achieved / FP64_PEAK_TFLOPS if "fp64" in info["pipe"] else None,
            "dmma_peak": DMMA_PEAK_TFLOPS,
            "frac_of_dmma_peak": achieved / DMMA_PEAK_TFLOPS if "DMMA" in info["pipe"] else None,
            "implemented_tflops": info.get("implemented_tflops"),
            "i8_peak_tops": I8_PEAK_TOPS if "i8" in info["pipe"] else None,
            "implemented_frac_of_i8_peak": (info["implemented_tflops"] / I8_PEAK_TOPS
                                            if "i8" in info["pipe"]
                                            and info.get("implemented_tflops") else None),
            "implemented_frac_of_dmma_peak": (info["implemented_tflops"] / DMMA_PEAK_TFLOPS
                                              if "DMMA" in info["pipe"]
                                              and info.get("implemented_tflops") else None),
            "note": ("float64 kernel: the bf16 tensor peak is not its ceiling; the measured "
                     "float64 tensor-core (DMMA) peak is" if "fp64" in info["pipe"] else
                     "float64-exact projection from int8 digits: `achieved` counts the "
                     "reference's 2p^2 flop per signal; the int8 ops it issues "
                     "(implemented_tflops, in TOPS) are rated against the measured kind::i8 "
                     "peak" if "i8" in info["pipe"] else None),
            "pipe": info["pipe"], "launches_per_step": info["launches"] / steps,
            "ms_per_step": info["ms_total"] / steps,
            "algorithmic": f"{info['flop_per_unit']} flop per unit, {info['units'] // steps} "
                           "units per step (DESIGN.md)"}


def iteration_model(p, K, s0, R, w_frac):
    """SURVEY.md §8(d) algorithmic FLOPs and bytes per signal of one iteration."""
    flops = 2 * p * p * (K + R) + 2 * p * s0 * R + w_frac * (2 * p * p * (R + 1) + 2 * p * s0 * R)
    bytes_ = 4 * p * (R + 2) + 4 * p * (R + 1) * w_frac + 4 * (10 + 5 * s0)
    return flops, bytes_


# --------------------------------------------------------------------------- CPU
def cpu_iteration_sample(a, y_rows, blocks, workers, iters=1, warm=1):
    """Time the reference algorithm (oracle port) on a bounded sample of the workload:
    mean seconds of ``iters`` iterations after ``warm`` untimed iterations."""
    from oracle import sbo_oracle as O
    y = y_rows.T.astype(np.float64)
    p, m = y.shape
    rep0 = O.code_signals(y, blocks, a.s0, workers=workers)
    w = max(p, m // 16)
    times = []
    for i in range(iters + warm):
        t0 = time.perf_counter()
        O.iterate(y, blocks, rep0.residual_sq, a.s0, a.rounds, w, seed=1, workers=workers)
        if i >= warm:
            times.append(time.perf_counter() - t0)
    return float(np.mean(times))


def cpu_sample_note(a, n, workers, t):
    """The cpu_baseline description, with the linear extrapolation to the full job."""
    return {"sample": (f"one iteration on the first {n} signals of the workload (p={a.p_edge**2}, "
                       f"K={a.K - 1}->{a.K}, s0={a.s0}, R={a.rounds}, W=m/16), oracle port: "
                       f"numpy/OpenBLAS 1 thread + a {workers}-thread pool, same entering "
                       "blocks"),
            "extrapolated_s_per_iteration_at_m_total": t * a.m_total / n,
            "extrapolation": (f"linear in m from the {n}-signal sample to m={a.m_total} "
                              "(SURVEY.md 8(d)); the CPU per-signal rate falls as m grows "
                              "(SURVEY.md 3.5), so this favours the CPU")}


def run_reference(a):
    """--impl reference: the reference algorithm on the host cores (rank 0 only).

    Each step is one iteration over a --cpu-sample (2^20) sample of the workload;
    the timed count is min(--steps, --cpu-steps) after min(--warmup, 1) warm-up
    iterations, so the arm ends within a few minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import sbo_oracle as O
    from paper_1412_4944_b200 import signals
    workers = os.cpu_count() or 1
    grid = signals.scene(a.scene, a.scene, 0)
    n = min(a.cpu_sample, a.m_total)
    rows = signals.unit_range(signals.patch_bytes(grid, a.p_edge, a.m_total, 11, 0, n))
    y = rows.T.astype(np.float64)
    p, m = y.shape
    blocks = O.initial_blocks(y, a.s0, a.K - 1, 4096, a.rounds, seed=1, workers=workers)
    rep0 = O.code_signals(y, blocks, a.s0, workers=workers)
    w = max(p, m // 16)
    steps, warm = max(1, min(a.steps, a.cpu_steps)), min(a.warmup, 1)
    times = []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        O.iterate(y, blocks, rep0.residual_sq, a.s0, a.rounds, w, seed=1, workers=workers)
        if i >= warm:
            times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    v = m / t
    cpu = {"value": v, "unit": "signals/s", "cores": workers, "kind": "port"}
    cpu.update(cpu_sample_note(a, m, workers, t))
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "signals/s", "n_gpus": a.gpus, "steps": a.steps,
        "steps_timed": steps, "warmup": a.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": workload_name(a, a.gpus), "sample_m": m},
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "signals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------- GPU
KERNELS_PER_CALL = {"sbo_energy_pass": 1, "sbo_group": 4, "sbo_code_segments": 1, "sbo_cand_sort": 3,
                    "sbo_outer_segments": 1, "sbo_reduce_segments": 1, "sbo_polar": 2,
                    "sbo_gram": 3, "sbo_init_block": 1, "sbo_worst_set": 19, "sbo_sum": 2,
                    "sbo_key_histogram": 1, "sbo_worst_collect": 3, "sbo_frobenius_sq": 2,
                    "sbo_round_code_segments": 1, "sbo_outer_i8_segments": 2, "sbo_i8_scan": 1,
                    "sbo_y_digits": 1, "sbo_y_tiles": 1, "sbo_round_i8_segments": 2,
                    "sbo_gram_counted": 3, "sbo_chunk_segments": 1,
                    "sbo_tc_split_signals": 1, "sbo_tc_split_blocks": 1, "sbo_tc_energy": 1,
                    "sbo_tc_energy256": 1, "sbo_energy_recheck_cand": 1,
                    "sbo_coef_i8_segments": 2, "sbo_select_coded": 1,
                    "sbo_energy_recheck_i8": 2}


def kernels_per_call(name: str, p: int, K: int) -> int:
    """Kernel launches behind one ABI call (gpu_launches)."""
    if name == "sbo_polar" and p > 64:
        return 3 + 3 * 40  # init, 40 x (2 GEMMs + check), finish, the Jacobi fallback
    if name == "sbo_energy_recheck_pairs":
        return 2 + 4 * K   # lists, reduce; per block: segments, digits, projection, selection
    return KERNELS_PER_CALL.get(name, 1)


def max_over_ranks(x: float, dist, dev) -> float:
    """Max of a per-rank time over all ranks (NCCL on the device, gloo on the host)."""
    import torch
    if dist is None:
        return x
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_1412_4944_b200.engine import Comm, Engine, Signals, TorchComm, require_device
    from paper_1412_4944_b200.sbo import SboConfig, _block_rng, _init_into

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SBO_BENCH_ONE_GPU=1: every rank on cuda:0 over gloo — a functional check of the
    # multi-rank path when the box has one GPU (not a performance configuration)
    one_gpu = os.environ.get("SBO_BENCH_ONE_GPU", "0") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = require_device(local)
    comm = Comm()
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        comm = TorchComm()
    rows, m_total = shard_signals(a, rank, world)
    p = rows.shape[1]
    eng = Engine(Signals.from_rows(rows, dev), a.s0, k_cap=a.K, comm=comm, m_total=m_total)
    lo, hi = shard_range(a, rank, world)

    def local_cols(cols):
        sel = cols[(cols >= lo) & (cols < hi)]
        return sel - lo

    cfg = SboConfig(s0=a.s0, k0=a.K - 1, p0=4096, rounds=a.rounds, k_max=a.K, seed=1)
    _init_into(eng, cfg, m_total, local_cols if world > 1 else None)
    eng.represent_full()
    torch.cuda.synchronize()
    snap_blocks = eng.blocks.clone()
    st = eng.state
    snap = [t.clone() for t in (st.best, st.score, st.norm, st.residual, st.total)]
    K0 = eng.K
    draws = _block_rng(1, 1, K0).standard_normal((p + 8, p))
    w = max(p, m_total // 16)

    # the entering state of every step: blocks and assignment (Engine.snapshot)
    entering = eng.snapshot()

    def restore():
        eng.restore(entering)

    class Marks:
        def __init__(self):
            self.ev = []

        def mark(self):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.ev.append(e)

    for _ in range(a.warmup):
        restore()
        eng.iterate(w, a.rounds, draws)
    # the step (restore + iteration) is replayed as a CUDA graph, which removes the
    # host launch gaps: on one GPU, and sharded over NCCL (stream-ordered
    # collectives, member counts kept on the device); gloo runs eagerly
    use_graph = ((world == 1 or getattr(comm, "capturable", False))
                 and os.environ.get("SBO_BENCH_NO_GRAPH", "0") != "1")
    replay, graph_note = None, None
    if use_graph:
        draws_dev = torch.from_numpy(np.ascontiguousarray(draws)).to(dev)
        try:
            replay = eng.capture_iteration(entering, w, a.rounds, draws_dev)
        except Exception as e:  # eager steps instead; the line says why
            graph_note = f"capture failed, eager steps: {type(e).__name__}: {e}"[:300]
            replay = None
            torch.cuda.synchronize()
    # kernels of one step (ABI calls x kernels per call), counted on an eager step
    calls = {}
    orig = eng._call

    def counting(name, *args, **kw):
        calls[name] = calls.get(name, 0) + 1
        return orig(name, *args, **kw)

    eng._call = counting
    restore()
    eng.iterate(w, a.rounds, draws)
    eng._call = orig
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record()
    for _ in range(a.steps):
        if replay is not None:
            out = replay()
        else:
            restore()
            out = eng.iterate(w, a.rounds, draws)
    t_end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    # per-kernel and per-phase breakdown: a separate instrumented pass (CUDA events
    # around every ABI call and at the phase boundaries), not part of `value`
    eng.timer = []
    marks = []
    for _ in range(a.steps):
        restore()
        mk = Marks()
        eng.iterate(w, a.rounds, draws, timer=mk)
        marks.append(mk)
    torch.cuda.synchronize()
    elapsed = t_start.elapsed_time(t_end) / 1e3
    elapsed = max_over_ranks(elapsed, dist if world > 1 else None, dev)
    t_step = elapsed / a.steps
    value = m_total / t_step
    launches = a.steps * sum(kernels_per_call(n, p, a.K) * c for n, c in calls.items())
    hbm, bf16, src = peaks()
    kernels = kernel_families(eng.timer, p, min(a.s0, p))
    eng.timer = None
    rated = [(k, v) for k, v in kernels.items() if v["tflops"]] or list(kernels.items())
    dom = max(rated, key=lambda kv: kv[1]["ms_total"])
    for v in kernels.values():
        v["ms_per_step"] = v["ms_total"] / a.steps
    f_sig, b_sig = iteration_model(p, a.K, a.s0, a.rounds, 1.0 / 16)
    m_gpu = hi - lo  # the largest shard is rank 0's
    t_roof = max(f_sig * m_gpu / (bf16 / 2 * 1e12), b_sig * m_gpu / (hbm * 1e9))
    phases = np.mean([[mk.ev[i].elapsed_time(mk.ev[i + 1]) for i in range(4)] for mk in marks],
                     axis=0)

    # e2e: host buffers through the public engine API, copies inside the timed region
    e2e = e2e_ingest = None
    if not a.no_e2e:
        e2e = run_e2e(a, eng, rows, snap_blocks, snap, K0, w, draws, dist if world > 1 else None)
        e2e_ingest = run_e2e(a, eng, rows, snap_blocks, snap, K0, w, draws,
                             dist if world > 1 else None, ingest=shard_corners(a, rank, world))

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        workers = os.cpu_count() or 1
        n = min(a.cpu_sample, rows.shape[0])
        blocks = [q for q in snap_blocks[:K0].cpu().numpy()]
        t = cpu_iteration_sample(a, rows[:n], blocks, workers, warm=0)
        cpu = {"value": n / t, "unit": "signals/s", "cores": workers, "kind": "port"}
        cpu.update(cpu_sample_note(a, n, workers, t))
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "signals/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded procedural scene, 8x8 patches, float32 signals)",
        "config": {"workload": workload_name(a, world), "p": p, "K": a.K, "s0": a.s0,
                   "rounds": a.rounds, "m_total": m_total, "m_per_gpu": hi - lo, "W": w,
                   "scaling": a.scaling,
                   "l2": (f"inputs larger than L2 (fp32 signals {4 * p * (hi - lo) / 1e9:.2f} GB "
                          "per GPU > 126 MB L2)"),
                   "parallelism": f"column shards over {world} GPU(s), NCCL allreduce"},
        "clocks": clocks,
        "gpu_launches": launches,
        "cuda_graph": bool(replay is not None),
        "cuda_graph_note": graph_note,
        "phases_ms": {"worst+new_block": phases[0], "represent1": phases[1],
                      "group+retrain": phases[2], "represent2": phases[3]},
        "roofline": roofline_of(dom[0], dom[1], bf16, src, steps=a.steps),
        "kernels": {k: v for k, v in kernels.items() if v},
        "iteration_roofline": {"flop_per_signal": f_sig, "bytes_per_signal": b_sig,
                               "t_roof_ms": t_roof * 1e3, "frac": t_roof / t_step,
                               "model": "SURVEY.md 8(d): max(F/TF32 peak, B/HBM)"},
        "e2e": e2e,
        "e2e_ingest": e2e_ingest,
        "cpu_baseline": cpu,
        "rmse": out.rmse,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def shard_corners(a, rank, world):
    """This rank's patch corners (data.py:199-201 draws over the whole workload)."""
    from paper_1412_4944_b200 import data, signals
    grid = signals.scene(a.scene, a.scene, 0)
    r, c = data.patch_corners(a.scene, a.scene, a.p_edge, a.m_total, 11)
    lo, hi = shard_range(a, rank, world)
    return grid, r[lo:hi].astype(np.int32), c[lo:hi].astype(np.int32)


def run_e2e(a, eng, rows, snap_blocks, snap, K0, w, draws, dist, ingest=None):
    """Same metric through the host-buffer path: every step uploads its signals and
    entering state (from pinned host memory), runs the iteration, and reads the new
    dictionary, assignment and residuals back; every copy is inside the timed region.
    Step i+1's uploads run on a copy stream while step i computes, as a training loop
    over streamed data would: two device signal buffers and two device staging sets
    for the entering state (restored into the live state by a device copy at the
    step's start), and the outputs leave through a device staging set on a third
    stream, so no host transfer sits on the compute stream.

    ``ingest`` = (grid, rows, cols): the step's input is the 8-bit scene and this
    rank's int32 patch corners instead of the float32 signal matrix; the patches are
    extracted on the device at the start of the step (data.extract_rows, the
    device form of data.py:182-208)."""
    import torch
    from paper_1412_4944_b200 import data as D
    st = eng.state
    if ingest is None:
        host_in = [torch.from_numpy(rows).pin_memory()]
    else:
        host_in = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in ingest]
    host_blocks = snap_blocks[:K0].cpu().pin_memory()
    # the entering state the iteration reads: best, score, residual, total (the
    # signal norms, snap[2], are not read by it and stay on the device)
    up_idx = (0, 1, 3, 4)
    host_state = [snap[i].cpu().pin_memory() for i in up_idx]
    host_draws = torch.from_numpy(np.ascontiguousarray(draws, dtype=np.float64)).pin_memory()
    out_blocks = torch.empty((K0 + 1,) + tuple(snap_blocks.shape[1:]), dtype=torch.float64).pin_memory()
    out_best = torch.empty(rows.shape[0], dtype=torch.int32).pin_memory()
    out_res = torch.empty(rows.shape[0], dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host_in) + host_blocks.numel() * 8 + \
        sum(t.numel() * t.element_size() for t in host_state)
    h2d += host_draws.numel() * 8  # the new block's completion draws
    d2h = out_blocks.numel() * 8 + out_best.numel() * 4 + out_res.numel() * 8
    # all on created streams: work on the legacy default stream would serialise
    # with the copy streams
    compute = torch.cuda.Stream(eng.dev)
    copier = torch.cuda.Stream(eng.dev)
    reader = torch.cuda.Stream(eng.dev)
    ybuf = [eng.sig.y, torch.empty_like(eng.sig.y)]
    dev_in = [ybuf[:1], [ybuf[1]]] if ingest is None else \
        [[torch.empty_like(t, device=eng.dev) for t in host_in] for _ in range(2)]
    entering = eng.snapshot()
    stg = [entering, {"K": K0, "exact_scores": True, "blocks": entering["blocks"].clone(),
                      "state": [t.clone() for t in entering["state"]]}]
    for sg in stg:
        sg["K"], sg["exact_scores"] = K0, True
    dev_draws = [torch.empty(host_draws.shape, dtype=torch.float64, device=eng.dev)
                 for _ in range(2)]
    out_dev = [torch.empty((K0 + 1,) + tuple(snap_blocks.shape[1:]), dtype=torch.float64,
                           device=eng.dev), torch.empty_like(st.best), torch.empty_like(st.residual)]
    ready = [torch.cuda.Event(), torch.cuda.Event()]   # step j's inputs are on the device
    freed = [None, None]                               # the last step using set j is done
    read_done = [None]                                 # out_dev is free again

    def upload(j):
        """Entering state + signals of a step into set j (copy stream)."""
        with torch.cuda.stream(copier):
            if freed[j] is not None:
                copier.wait_event(freed[j])
            stg[j]["blocks"][:K0].copy_(host_blocks, non_blocking=True)
            for i, src in zip(up_idx, host_state):
                stg[j]["state"][i].copy_(src, non_blocking=True)
            dev_draws[j].copy_(host_draws, non_blocking=True)
            for dst, src in zip(dev_in[j], host_in):
                dst.copy_(src, non_blocking=True)
            ready[j].record(copier)

    def device_step(j):
        eng.restore(stg[j])
        if ingest is not None:  # patches of the uploaded scene, on the device
            g, r, c = dev_in[j]
            D.extract_rows(g, D.GRID_U8, a.p_edge, r, c, "unit-range", out=ybuf[j],
                           stream=eng.stream)
        eng.refresh_signals(rescan=False)  # operand split + digit rows of the new signals
        return eng.iterate_device(w, a.rounds, dev_draws[j])

    # one GPU: each set's step (restore + operand split + iteration) as a CUDA graph
    graphs = [None, None]
    if dist is None and os.environ.get("SBO_BENCH_NO_GRAPH", "0") != "1":
        for j in range(2):
            stg[j]["blocks"][:K0].copy_(host_blocks.to(eng.dev))
            for i, src in zip(up_idx, host_state):
                stg[j]["state"][i].copy_(src.to(eng.dev))
            dev_draws[j].copy_(host_draws.to(eng.dev))
            for dst, src in zip(dev_in[j], host_in):
                dst.copy_(src.to(eng.dev))
            eng.sig.y = ybuf[j]
            graphs[j] = eng.capture(lambda j=j: device_step(j), lambda: None)
        eng.sig.y = ybuf[0]

    def step(j):
        compute.wait_event(ready[j])
        eng.sig.y = ybuf[j]
        eng.K = K0
        if graphs[j] is not None:
            graphs[j][0].replay()
            out = graphs[j][1]
        else:
            out = device_step(j)
        freed[j] = torch.cuda.Event()
        freed[j].record(compute)
        if read_done[0] is not None:
            compute.wait_event(read_done[0])
        out_dev[0].copy_(eng.blocks[: K0 + 1])
        out_dev[1].copy_(st.best)
        out_dev[2].copy_(st.residual)
        staged = torch.cuda.Event()
        staged.record(compute)
        with torch.cuda.stream(reader):
            reader.wait_event(staged)
            for dst, src in zip((out_blocks, out_best, out_res), out_dev):
                dst.copy_(src, non_blocking=True)
            read_done[0] = torch.cuda.Event()
            read_done[0].record(reader)
        eng.finish_iteration(out)

    torch.cuda.synchronize()
    with torch.cuda.stream(compute):
        upload(0)
        step(0)  # warm-up
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(compute)
        copier.wait_event(s)
        upload(0)
        dbg = os.environ.get("SBO_E2E_DEBUG") == "1"
        for i in range(a.steps):
            t0 = time.perf_counter()
            if i + 1 < a.steps:
                upload((i + 1) % 2)  # overlaps step i
            t1 = time.perf_counter()
            step(i % 2)
            if dbg:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(compute)
                ev.synchronize()
                print(f"e2e step {i}: issue {1e3 * (t1 - t0):.2f} ms, step {1e3 * (time.perf_counter() - t1):.2f} ms, "
                      f"since start {s.elapsed_time(ev):.2f} ms", file=sys.stderr)
        compute.wait_event(read_done[0])  # the last step's results are on the host
        e.record(compute)
    torch.cuda.synchronize()
    eng.sig.y = ybuf[0]
    t = max_over_ranks(s.elapsed_time(e) / 1e3 / a.steps, dist, eng.dev)
    m_total = eng.m_total
    out = {"value": m_total / t, "unit": "signals/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h,
           "pipelining": "step i+1's input and state uploads overlap step i (copy stream); "
                         "results leave through a device staging copy on a third stream",
           "api": ("the sbo_train loop body through Engine (restore entering state, "
                   "iterate_device, finish_iteration) with host buffers; the new dictionary, "
                   "assignment and residuals are read back (codes and energies stay on the "
                   "device), not the sbo_train/represent entry points themselves")}
    if ingest is not None:
        out["input"] = ("8-bit scene + int32 patch corners per step; patches extracted on the "
                        "device (paper_1412_4944_b200.data, data.py:182-208)")
    return out


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(a)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
