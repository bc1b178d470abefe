"""Several logical workers of one process stepped in lockstep on one device.

The reference runs its workers as threads that meet at one spin barrier per step
(/root/reference/pkg/src/mpmbench/bench.py:334-370, multiworker.py:27-70).  Work before the
barrier touches only worker-local state, so running "pre-barrier phase of every worker, then
post-barrier phase of every worker" on one CUDA stream is the same schedule with the barrier
realised by stream order.  This is how the cross-worker halo reduction (peer rows read inside
the grid-update kernel) is exercised on a single GPU; with one process per GPU the same
worker code runs under `DistRuntime` (dist.py).

Populations: `material` may be a sequence with one Material per worker.  Each worker then
carries one material population (its own constitutive kernel instantiation and channel
count) and the populations meet on the grid exactly as spatial partitions do -- mass and
momentum rows of blocks present in several tables are summed in the grid update
(pipeline.py:1172-1188).  This is how mixed snow / sand scenes (BASELINE.json configs[4]) run;
the reference itself has one material per run.
"""
from __future__ import annotations

import numpy as np
import torch

from .domain import cfl_dt
from .errors import ConfigError
from .multiworker import SharedRuntime, partition_particles
from .options import PipelineOptions
from .worker import CudaWorker


class CudaCluster:
    def __init__(self, n, params, material, boundary, options=None, initial_vmax=0.0, device=None,
                 **worker_kw):
        self.runtime = SharedRuntime(n, initial_vmax=initial_vmax)
        options = options if options is not None else PipelineOptions()
        materials = list(material) if isinstance(material, (list, tuple)) else [material] * n
        if len(materials) != n:
            raise ConfigError(f"{n} workers need {n} materials, got {len(materials)}")
        self.workers = [CudaWorker(w, self.runtime, params, materials[w], boundary, options,
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

    def seed_populations(self, populations):
        """One population per worker: (positions, velocities, mass) or (positions, velocities,
        mass, ids).  Ids default to consecutive ranges in population order."""
        if len(populations) != len(self.workers):
            raise ConfigError(f"{len(self.workers)} workers need {len(self.workers)} populations")
        base = 0
        for w, pop in zip(self.workers, populations):
            pos, vel, mass = pop[0], pop[1], pop[2]
            n = len(pos)
            ids = np.asarray(pop[3], dtype=np.int64) if len(pop) > 3 else np.arange(base, base + n, dtype=np.int64)
            if n:
                w.seed_particles(pos, vel, mass, ids=ids)
            base += n

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
            c_sound = max(w.material.sound_speed() for w in ws)
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
        nch = max(c[0].shape[1] for c in chunks)      # populations may differ in channel count
        chunks = [(np.pad(c[0], ((0, 0), (0, nch - c[0].shape[1]))), c[1]) for c in chunks]
        flat = np.concatenate([c[0] for c in chunks], axis=0)
        ids = np.concatenate([c[1] for c in chunks], axis=0)
        return flat[np.argsort(ids, kind="stable")]

    def positions_sorted_by_id(self):
        return self.state_sorted_by_id()[:, :3]
