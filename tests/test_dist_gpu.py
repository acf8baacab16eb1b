"""The signal-sharded iteration end to end on real kernels: two ranks (gloo, both
on cuda:0 — the pool gives one GPU per run) each own half of the signals, and one
iteration must reproduce the single-process engine: the same worst set, the same
assignment, and blocks equal to float64 summation-order differences (the P
allreduce adds the two ranks' partials in a different order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind="gaussian"):
    """Gaussian rows (the float64 DMMA rounds) or unit-range patches (the
    integer-digit tcgen05 rounds, round_i8.cu / outer_i8.cu)."""
    from paper_1412_4944_b200 import signals
    rng = np.random.default_rng(77)
    p, K = 64, 4
    y32 = (signals.gaussian_signals(p, 16384, seed=9) if kind == "gaussian"
           else signals.patch_signals(16384, 8, 512, 512))
    blocks = np.stack([np.linalg.qr(rng.standard_normal((p, p)))[0] for _ in range(K)])
    return y32, blocks


def _run_rank(rank, world, port, out, kind):
    import torch.distributed as dist

    from paper_1412_4944_b200 import dist as D
    from paper_1412_4944_b200.engine import Engine, Signals, TorchComm, require_device
    from paper_1412_4944_b200.sbo import _block_rng
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = require_device(0)
        y32, blocks = _problem(kind)
        m = y32.shape[0]
        lo, hi = D.shard_range(m, world, rank)
        eng = Engine(Signals.from_rows(y32[lo:hi], dev), 8, k_cap=len(blocks) + 1,
                     comm=TorchComm(), m_total=m)
        eng.set_blocks(blocks)
        eng.represent_full()
        draws = _block_rng(0, 1, len(blocks)).standard_normal((72, 64))
        res = eng.iterate(m // 16, 3, draws)
        out[rank] = (eng.blocks[: eng.K].cpu().numpy(), res.rmse,
                     res.worst.cpu().numpy().astype(np.int64) + lo,
                     eng.state.best.cpu().numpy(), eng.state.residual.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["gaussian", "patches"])
def test_two_ranks_match_single_process(kind):
    from paper_1412_4944_b200.engine import Engine, Signals, require_device
    from paper_1412_4944_b200.sbo import _block_rng
    dev = require_device(0)
    y32, blocks = _problem(kind)
    m = y32.shape[0]
    eng = Engine(Signals.from_rows(y32, dev), 8, k_cap=len(blocks) + 1)
    eng.set_blocks(blocks)
    eng.represent_full()
    draws = _block_rng(0, 1, len(blocks)).standard_normal((72, 64))
    ref = eng.iterate(m // 16, 3, draws)
    ref_blocks = eng.blocks[: eng.K].cpu().numpy()
    ref_best = eng.state.best.cpu().numpy()
    ref_res = eng.state.residual.cpu().numpy()
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_run_rank, args=(r, 2, port, out, kind)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=600)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    b0, rmse0, w0, best0, res0 = out[0]
    b1, rmse1, w1, best1, res1 = out[1]
    np.testing.assert_array_equal(b0, b1)  # identical reduced P -> identical blocks per rank
    assert np.abs(b0 - ref_blocks).max() < 1e-9
    np.testing.assert_array_equal(np.sort(np.concatenate([w0, w1])),
                                  np.sort(ref.worst.cpu().numpy()))
    np.testing.assert_array_equal(np.concatenate([best0, best1]), ref_best)
    np.testing.assert_allclose(np.concatenate([res0, res1]), ref_res, rtol=1e-9, atol=1e-12)
    assert rmse0 == rmse1 and rmse0 == pytest.approx(ref.rmse, rel=1e-12)


def test_nccl_sharded_step_captured_as_graph():
    """The sharded code path on NCCL (one rank: the pool gives one GPU; the
    collectives still run through NCCL): the worst set's member count stays on
    the device, so the whole step is captured as one CUDA graph, and replays
    equal both the eager sharded step and the single-GPU engine."""
    import torch.distributed as dist

    from paper_1412_4944_b200.engine import Engine, Signals, TorchComm, require_device
    from paper_1412_4944_b200.sbo import _block_rng
    dev = require_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        y32, blocks = _problem("patches")
        m = y32.shape[0]
        draws = _block_rng(0, 1, len(blocks)).standard_normal((72, 64))
        outs = []
        for comm in (None, TorchComm(sharded=True)):
            eng = Engine(Signals.from_rows(y32, dev), 8, k_cap=len(blocks) + 1, comm=comm,
                         m_total=m)
            eng.set_blocks(blocks)
            eng.represent_full()
            snap = eng.snapshot()
            res = eng.iterate(m // 16, 3, draws)
            outs.append((eng.blocks[: eng.K].cpu().numpy(), eng.state.best.cpu().numpy(),
                         res.rmse, np.sort(res.worst.cpu().numpy())))
            if comm is not None:
                assert comm.capturable
                replay = eng.capture_iteration(snap, m // 16, 3,
                                               torch.from_numpy(draws).to(dev))
                for _ in range(2):
                    r2 = replay()
                    outs.append((eng.blocks[: eng.K].cpu().numpy(),
                                 eng.state.best.cpu().numpy(), r2.rmse,
                                 np.sort(r2.worst.cpu().numpy())))
        ref = outs[0]
        for b, best, rmse, worst in outs[1:]:
            np.testing.assert_array_equal(best, ref[1])
            np.testing.assert_array_equal(worst, ref[3])
            assert np.abs(b - ref[0]).max() < 1e-12
            assert rmse == pytest.approx(ref[2], rel=1e-13)
    finally:
        dist.destroy_process_group()
