"""Worker-count knobs of the reference executor (parallel.py:13-54), kept for API parity.

The reference parallelizes with a thread pool over fixed 256-column tiles and
guarantees results independent of the worker count.  Here the parallel
decomposition is the CUDA grid (and the rank count for sharded runs); the
``workers`` / ``ORTHODICT_WORKERS`` knob is validated exactly like the reference
and otherwise has no effect on results — the same contract, trivially kept.
"""
from __future__ import annotations

import os

WORKERS_ENV = "ORTHODICT_WORKERS"


def resolve_workers(workers: int | None = None) -> int:
    """Explicit count, else ORTHODICT_WORKERS, else the CPU count (parallel.py:16-29)."""
    if workers is None:
        env = os.environ.get(WORKERS_ENV)
        if env is not None:
            try:
                workers = int(env)
            except ValueError:
                raise ValueError(f"{WORKERS_ENV} must be an integer, got {env!r}") from None
        else:
            workers = os.cpu_count() or 1
    if workers < 1:
        raise ValueError(f"worker count must be at least 1, got {workers}")
    return workers
