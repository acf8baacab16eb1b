"""bench.py's command line: `--gpus N` re-launches the script under
torch.distributed.run, whose own parser sees every argument first — each bench
option must reach the script unchanged (an option that is a prefix of a
launcher option, like the former `--m`, made the launcher exit)."""
import sys

import pytest

import bench


ARGV = ["--gpus", "2", "--steps", "3", "--warmup", "3", "--impl", "ours",
        "--m-total", "1048576", "--m-per-gpu", "524288", "--p-edge", "8", "--K", "16",
        "--s0", "8", "--rounds", "6", "--scene", "4096", "--cpu-sample", "65536",
        "--cpu-steps", "1", "--no-cpu-baseline", "--no-e2e"]


def test_relaunch_keeps_every_bench_option():
    run = pytest.importorskip("torch.distributed.run")
    args = run.get_args_parser().parse_args(bench.relaunch_args(2, 29500, ARGV))
    assert args.nproc_per_node == "2"
    assert args.training_script.endswith("bench.py")
    assert args.training_script_args == ARGV


def test_bench_parses_the_same_options(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"] + ARGV)
    a = bench.parse()
    assert (a.gpus, a.steps, a.warmup, a.K, a.s0, a.rounds) == (2, 3, 3, 16, 8, 6)
    assert a.scaling == "weak" and a.no_e2e and a.no_cpu_baseline


def test_defaults_are_config_c(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert bench.config_label(a) == "C" and a.scaling == "strong" and a.warmup >= 3
