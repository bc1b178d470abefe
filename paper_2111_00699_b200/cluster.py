"""Several logical workers of one process stepped in lockstep on one device.

The reference runs its workers as threads that meet at one spin barrier per step
(/root/reference/pkg/src/mpmbench/bench.py:334-370, multiworker.py:27-70).  Work before the
barrier touches only worker-local state, so running "pre-barrier phase of every worker, then
post-barrier phase of every worker" on one CUDA stream is the same schedule with the barrier
realised by stream order.  This is how the cross-worker halo reduction (peer rows read inside
the grid-update kernel) is exercised on a single GPU; with one process per GPU the same
worker code runs under `DistRuntime` (dist.py).
"""
from __future__ import annotations

import numpy as np
import torch

from .domain import cfl_dt
from .multiworker import SharedRuntime, partition_particles
from .options import PipelineOptions
from .worker import CudaWorker


class CudaCluster:
    def __init__(self, n, params, material, boundary, options=None, initial_vmax=0.0, device=None,
                 **worker_kw):
        self.runtime = SharedRuntime(n, initial_vmax=initial_vmax)
        options = options if options is not None else PipelineOptions()
        self.workers = [CudaWorker(w, self.runtime, params, material, boundary, options,
                                   device=device, **worker_kw) for w in range(n)]
        self.params = params
        self.cfl_mode = False
        self.frame_steps = 0

    def seed(self, positions, velocities, mass):
        """bench.py:434-439: partition along the longest axis, ids = original indices."""
        positions = np.asarray(positions)
        velocities = np.asarray(velocities)
        parts = partition_particles(positions, len(self.workers))
        for w, part in zip(self.workers, parts):
            if len(part):
                w.seed_particles(positions[part], velocities[part], mass, ids=part)
        return parts

    def run_step(self, step):
        for w in self.workers:
            w.step_pre_barrier(step)
        self.runtime.generations += 1      # the one barrier of the step (pipeline.py:931)
        for w in self.workers:
            w.step_post_barrier(step)

    def run_frame(self):
        ws = self.workers
        self.frame_steps = 0
        for w in ws:
            w.begin_frame()
        if self.cfl_mode:
            c_sound = ws[0].material.sound_speed()
            t = 0.0
            while t < self.params.frame_dt - 1e-12:
                vmax = self.runtime.global_vmax((ws[0]._global_step - 2) % 3)
                dt = cfl_dt(vmax + c_sound, self.params, self.params.frame_dt - t)
                for w in ws:
                    w.dt = dt
                self.run_step(ws[0]._global_step)
                t += dt
                self.frame_steps += 1
        else:
            for w in ws:
                w.dt = self.params.dt
            for _ in range(self.params.steps_per_frame):
                self.run_step(ws[0]._global_step)
                self.frame_steps += 1
        for w in ws:
            if w._pending_gather:
                w._flush_gather()

    def state_sorted_by_id(self):
        chunks = [w.store.state_with_ids() for w in self.workers]
        flat = np.concatenate([c[0] for c in chunks], axis=0)
        ids = np.concatenate([c[1] for c in chunks], axis=0)
        return flat[np.argsort(ids, kind="stable")]

    def positions_sorted_by_id(self):
        return self.state_sorted_by_id()[:, :3]
