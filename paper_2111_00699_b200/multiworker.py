"""Cross-worker state and partitioning (host side).

Mirrors /root/reference/pkg/src/mpmbench/multiworker.py:73-137.  In the reference the
workers are threads that meet at a spin barrier; here a worker is a GPU (one process per GPU
under torch.distributed, or several logical workers of one process on one device for tests)
and the "barrier" is stream order / the collective that exchanges the halo rows.  The
publication slots keep the reference's shape: per-parity step records and a 3-slot vmax ring.
"""
from __future__ import annotations

import numpy as np

from .errors import RejectedInputError


class SharedRuntime:
    """In-process runtime for `n_workers` logical workers (multiworker.py:73-107)."""

    def __init__(self, n_workers: int, barrier_timeout: float = 10.0, initial_vmax: float = 0.0):
        if n_workers < 1:
            raise RejectedInputError(f"barrier needs >= 1 workers, got {n_workers}")
        self.n_workers = n_workers
        self.barrier_timeout = barrier_timeout
        self.generations = 0
        self._steps = [[None] * n_workers, [None] * n_workers]
        self._vmax = np.full((3, n_workers), float(initial_vmax))

    def seed_vmax(self, value: float) -> None:
        self._vmax[:, :] = float(value)

    def barrier_wait(self, worker_id: int) -> int:
        """Single-worker runtimes pass straight through; several logical workers are stepped
        in lockstep phases by CudaCluster, which counts the generation itself."""
        if self.n_workers == 1:
            self.generations += 1
        return self.generations

    def publish_step(self, parity: int, worker_id: int, state) -> None:
        self._steps[parity & 1][worker_id] = state

    def peer_step(self, parity: int, worker_id: int):
        return self._steps[parity & 1][worker_id]

    def publish_vmax(self, slot: int, worker_id: int, value: float) -> None:
        self._vmax[slot % 3, worker_id] = value

    def global_vmax(self, slot: int) -> float:
        return float(self._vmax[slot % 3].max())


def partition_particles(positions, n: int):
    """n near-equal contiguous index ranges along the longest bounding-box axis
    (multiworker.py:114-137): stable argsort, remainder handed out from worker 0."""
    if n < 1:
        raise RejectedInputError(f"worker count must be >= 1, got {n}")
    pos = np.asarray(positions, dtype=np.float64)
    count = pos.shape[0]
    if count == 0:
        return [np.empty(0, dtype=np.int64) for _ in range(n)]
    extent = pos.max(axis=0) - pos.min(axis=0)
    axis = int(np.argmax(extent))
    order = np.argsort(pos[:, axis], kind="stable")
    base, rem = divmod(count, n)
    out, start = [], 0
    for w in range(n):
        s = base + 1 if w < rem else base
        out.append(order[start:start + s])
        start += s
    return out


class EfficiencyReport:
    """Multi-worker scaling: e = t1 / (n * tn), 1.0 is ideal (multiworker.py:191-211)."""

    def __init__(self, t1_ms: float, tn_ms: float, n: int):
        if t1_ms <= 0.0 or tn_ms <= 0.0:
            raise RejectedInputError(f"timings must be positive, got t1={t1_ms} tn={tn_ms}")
        if n < 1:
            raise RejectedInputError(f"worker count must be >= 1, got {n}")
        self.t1_ms, self.tn_ms, self.n = t1_ms, tn_ms, n
        self.e = t1_ms / (n * tn_ms)
        self.anomalous = self.e > 1.05


def efficiency(t1_ms: float, tn_ms: float, n: int) -> EfficiencyReport:
    return EfficiencyReport(t1_ms, tn_ms, n)
