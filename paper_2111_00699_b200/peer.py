"""One process per GPU, halo rows read in place over NVLink, device-paced steps.

`DistWorker` (dist.py) follows the reference's protocol literally: one host collective per step
(the barrier), halo rows packed and exchanged with send/recv.  At eight GPUs a substep of the
1.33 M-particle scene is tens of microseconds of kernel time, so a host round trip per step is
the bound.  `PeerDistWorker` keeps the reference's data flow (pipeline.py:1166-1188: after the
step's one barrier every worker adds its peers' raw rows of the shared blocks) but moves the
barrier and the exchange onto the devices, the way the paper does it (PAPER.md:393,548-551:
peers' nodal rows are read through NVLink inside the grid kernel, interior blocks overlap):

  memory    every rank maps the others' raw[2], touched[2] and a small mailbox (CUDA IPC via
            torch's tensor reductions; re-exchanged only when a buffer was reallocated);
  signal    after the scatter of step s a rank stores s + 1 to its mailbox word
            (mpm_signal_step, release at system scope);
  wait+sum  mpm_grid_update spins on the peers' words (acquire, system scope) in the CTAs that
            own shared blocks -- and in CTA 0, which makes the kernel a full barrier -- then adds
            the peers' rows straight from their HBM; interior CTAs never wait;
  guard     the "rebuild needed" guard word of the speculative pipeline (worker.py) is
            replicated: the gather that raises it raises every rank's copy (system-scope
            atomicMin) before its rank signals, so all ranks stop after the same step;
  host      enqueues `depth` steps ahead and only reads status blocks; host collectives happen
            on the first step of a frame and on rebuild steps (code lists, re-tagging of the
            shared blocks, remapping), never on a steady-state step.

Raw rows alternate by step parity exactly as in the reference (pipeline.py:10-14): a rank
clears raw[par] at step s + 2, after its grid update of step s + 1 has waited for every peer's
signal of step s + 1, which those peers issue after their own grid update of step s -- the
read of raw[par] at step s is therefore complete.

With `lazy_flush=True` (worker.py) a frame may end with the fused gather pending; the next
frame then starts device-paced as well (no per-frame host collective).  Reading the particle
store completes the gather and makes the next frame start with a collective step, so store
reads must be SPMD (every rank or none).

The same sequence of steps and rebuilds as the reference results (tests/dist_check.py compares
against the reference's two-worker dump).  CFL-auto frames need the global max speed on the host
every step and use collective (host-paced) steps throughout.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from .dist import DistRuntime, DistWorker
from .errors import BarrierTimeoutError, ContractViolationError, ResourceError
from .memory import DeviceBuffer
from .worker import _INT_MAX, _RING, _stream_ptr

MAILBOX_WORDS = 16
MB_STEP, MB_GUARD, MB_WAIT_ERR = 0, 1, 2

SKIPPED, DONE, RAISED = 0, 1, 2


class PeerRuntime(DistRuntime):
    """DistRuntime + mapping of the other ranks' device buffers into this process."""

    def host_barrier(self):
        self.all_gather_i64([0])

    def probe(self) -> bool:
        """Collective.  True when every rank can map every other rank's device memory and read
        it from its own device (CUDA IPC + peer access): what PeerDistWorker relies on.  A caller
        falls back to the send/recv transport (dist.py) when this says no."""
        mine = torch.full((16,), self.wid + 1, dtype=torch.int32, device=self.device)
        torch.cuda.synchronize(self.device)
        ok = 1
        try:
            mem = self.exchange_tensors({"probe": mine})
        except Exception:
            mem, ok = None, 0
        if mem is not None:
            lib = _capi.lib()
            for q, m in enumerate(mem):
                if q == self.wid:
                    continue
                word = C.c_int32(0)
                if lib.mpm_peek_i32(m["probe"].data_ptr(), C.byref(word)) != 0 or word.value != q + 1:
                    ok = 0
        self._probe_keepalive = mine
        return bool(self.all_gather_i64([ok])[:, 0].all())

    def exchange_tensors(self, named: dict):
        """Collective.  Returns one dict per rank of objects with .data_ptr() addressing THAT
        rank's device memory from this rank's device (this rank's own entry holds the tensors
        passed in).

        The exporter's side is torch's storage sharing (cudaIpcGetMemHandle of the caching
        allocator's block + the offset inside it); the importer opens the handle itself
        (mpm_ipc_open) in ITS OWN device context with lazy peer access.  torch's own rebuild
        (torch.multiprocessing.reductions) maps the block in a context of the exporting device,
        which is what a tensor living "on cuda:q" needs, but not what a kernel running on this
        rank's GPU needs: that takes a mapping (and peer access) in this rank's context."""
        try:
            payload = self._export_payload(named)
        except Exception as exc:            # stay in step with the other ranks: fail after the collective
            payload, failure = None, exc
        gathered = [None] * self.n_workers
        dist.all_gather_object(gathered, payload, group=self.group)
        if any(pl is None for pl in gathered):
            raise ResourceError("a rank could not export its device buffers over CUDA IPC"
                                + (f": {failure}" if payload is None else ""))
        lib = _capi.lib()
        out = []
        for q, pl in enumerate(gathered):
            if q == self.wid:
                out.append(dict(named))
                continue
            mem = {}
            for k, (handle, offset, nbytes) in pl.items():
                base = self._ipc_open.get((q, handle))
                if base is None:
                    ptr = C.c_void_p()
                    _capi.check(lib.mpm_ipc_open(handle, C.byref(ptr)), "mpm_ipc_open")
                    base = self._ipc_open[(q, handle)] = int(ptr.value)
                mem[k] = MappedMemory(base + offset, nbytes)
            out.append(mem)
        return out

    @staticmethod
    def _export_payload(named: dict):
        payload = {}
        for k, t in named.items():
            st = t.untyped_storage()
            _, handle, _, block_offset = st._share_cuda_()[:4]
            handle = bytes(handle)
            if len(handle) in (65, 66):
                # recent caching allocators prefix the 64-byte cudaIpcMemHandle_t with [a version
                # byte and] a type tag: 'c' = cudaMalloc block; expandable segments ('e') are
                # shared as file descriptors
                if handle[-65:-64] != b"c":
                    raise ResourceError("peer-mapped halo rows need cudaMalloc-backed torch blocks "
                                        "(PYTORCH_CUDA_ALLOC_CONF=expandable_segments must be off)")
                handle = handle[-64:]
            if len(handle) != 64:
                raise ResourceError(f"unexpected CUDA IPC handle of {len(handle)} bytes")
            payload[k] = (handle, int(block_offset) + t.storage_offset() * t.element_size(),
                          t.numel() * t.element_size())
        return payload

    _ipc_open: dict = {}     # (rank, handle) -> base address in this process; process-wide, never closed
                             # while the group lives (the exporter's caching allocator keeps its blocks)


class MappedMemory:
    """A peer's buffer as seen from this rank's device."""
    __slots__ = ("ptr", "nbytes")

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = int(ptr), int(nbytes)

    def data_ptr(self) -> int:
        return self.ptr


class PeerDistWorker(DistWorker):
    def __init__(self, runtime: PeerRuntime, params, material, boundary, options=None,
                 wait_timeout_ms: int = 20000, depth: int = 2, **kw):
        super().__init__(runtime, params, material, boundary, options, **kw)
        with torch.cuda.device(self.device):
            self._mailbox = torch.zeros(MAILBOX_WORDS, dtype=torch.int32, device=self.device)
            self._mailbox[MB_GUARD] = _INT_MAX
            # the replicated guard word lives in memory the peers can reach
            self._guard_word = self._mailbox[MB_GUARD:MB_GUARD + 1]
            self._guard_host = torch.full((_RING,), _INT_MAX, dtype=torch.int32).pin_memory()
            self._guard_alias = self.lib.mpm_host_alias(self._guard_host.data_ptr())
        self.wait_timeout_ms = int(wait_timeout_ms)
        self.depth = max(1, int(depth))
        self._peer_mem = None
        self._exported_sig = None
        self._peer_counts = [0] * runtime.n_workers
        self._collective = False
        self.collective_steps = 0
        self.device_paced_steps = 0
        self.batched_steps = 0
        self._prof = None
        self._need_collective = True   # first step ever; after that only when some rank asks for it
        self.batch_steps = 4          # steps per mpm_enqueue_steps call (0 = one guarded step per call)

    # -- instrumentation of the device-side barrier / halo reads (off by default) -------------
    def enable_profile(self, on=True):
        """Counters kept by the grid update (mpm_grid_params.prof): barrier wait seen by CTA 0 and
        bytes of peer rows read.  `profile` reports them per launch."""
        with torch.cuda.device(self.device):
            self._prof = torch.zeros(8, dtype=torch.int64, device=self.device) if on else None

    @property
    def profile(self):
        if self._prof is None:
            return None
        p = self._prof.cpu().numpy()
        n = max(int(p[0]), 1)
        return {"grid_updates": int(p[0]), "barrier_wait_us_per_step": float(p[1]) / n / 1e3,
                "halo_bytes_per_step": float(p[2]) / n, "waiting_ctas_per_step": float(p[3]) / n}

    # -- exported memory -------------------------------------------------------------------
    def _exports(self):
        gr, tb = self.grid, self.table
        named = {"raw0": gr._raw[0].data, "raw1": gr._raw[1].data,
                 "touched0": tb._touched[0].data, "touched1": tb._touched[1].data,
                 "codes": tb._codes.data, "mailbox": self._mailbox}
        # a rank without blocks has nothing to map; peers never dereference its rows (count 0)
        return {k: (t if t.numel() else self._mailbox) for k, t in named.items()}

    def _export_sig(self):
        return tuple((t.data_ptr(), t.numel()) for t in self._exports().values())

    def _make_guard(self, step):
        g = _capi.Guard(self._guard_word.data_ptr(), step)
        k = 0
        if self._peer_mem is not None:
            for q, mem in enumerate(self._peer_mem):
                if q == self.runtime.wid:
                    continue
                g.peer_words[k] = mem["mailbox"].data_ptr() + 4 * MB_GUARD
                k += 1
        g.n_peer_words = k
        return g

    # -- step phases ------------------------------------------------------------------------
    def _publish(self, par, rebuilt):
        self._rebuilt_this_step = rebuilt
        # "my scatter of this step is complete": peers wait for it inside their grid update
        self._call("mpm_signal_step", self._mailbox.data_ptr() + 4 * MB_STEP, self._global_step + 1,
                   self._gref(), _stream_ptr())

    def _post_barrier(self, par):
        """Host collectives of a collective step: who rebuilt, remapping of reallocated buffers,
        re-tagging of the shared blocks (pipeline.py:1147-1164).  A device-paced step keeps the
        maps of the last collective step (no table changed since)."""
        if not self._collective:
            return
        rt, tb = self.runtime, self.table
        step = self._global_step
        any_rebuilt, counts = rt.step_info(step, self._rebuilt_this_step, tb.count)
        sig = self._export_sig()
        changed = rt.all_gather_i64([int(sig != self._exported_sig)])[:, 0].any()
        if changed or self._peer_mem is None:
            self._peer_mem = None        # drop the old mappings first
            self._peer_mem = rt.exchange_tensors(self._exports())
            self._exported_sig = sig
            self._guard = self._make_guard(step)
        self._peer_counts = list(counts)
        if not any_rebuilt:
            return
        # The peers' block-code lists are read where they lie (their tables are mapped like their
        # rows): every rank has passed the second host sync of its rebuild before it reached the
        # step_info exchange above, so the lists are complete in memory.
        stream = _stream_ptr()
        for q in range(rt.n_workers):
            if q == rt.wid:
                continue
            if tb.count == 0 or counts[q] == 0:
                self._peer_map[q] = None
                continue
            m = self._peer_map[q]
            if m is None:
                m = self._peer_map[q] = DeviceBuffer(torch.int32, (), self.device)
            m.resize(tb.count, keep=False)
            self._call("mpm_tag_shared", self._peer_mem[q]["codes"].data_ptr(), int(counts[q]), tb._hkeys.ptr,
                       tb._hvals.ptr, tb.hash_cap, m.ptr, tb.count, stream)

    def _fill_peers(self, gp, par=None, plan=None):
        """Peers' rows / flags / maps and the device-side barrier of a grid update.  With `plan`
        the rows of both parities go into the step plan (mpm_enqueue_steps picks per step)."""
        rt = self.runtime
        k = w = 0
        for q in range(rt.n_workers):
            if q == rt.wid:
                continue
            mem = self._peer_mem[q]
            gp.wait_flags[w] = mem["mailbox"].data_ptr() + 4 * MB_STEP
            w += 1
            if self._peer_map[q] is None or self._peer_counts[q] == 0:
                continue
            if plan is None:
                gp.peer_raw[k] = mem[f"raw{par}"].data_ptr()
                gp.peer_touched[k] = mem[f"touched{par}"].data_ptr()
            else:
                for pp in (0, 1):
                    plan.peer_raw[pp][k] = mem[f"raw{pp}"].data_ptr()
                    plan.peer_touched[pp][k] = mem[f"touched{pp}"].data_ptr()
            gp.peer_map[k] = self._peer_map[q].ptr
            k += 1
        gp.n_peers = k
        gp.n_wait = w
        gp.wait_timeout_ms = self.wait_timeout_ms
        gp.wait_error = self._mailbox.data_ptr() + 4 * MB_WAIT_ERR
        gp.block_filter = 0
        gp.fuse_clear = 0
        gp.prof = self._prof.data_ptr() if self._prof is not None else None

    def _reduce_and_update(self, par, step=None):
        if step is None:
            step = self._global_step
        tb = self.table
        gp = self._grid_params()
        self._fill_peers(gp, par)
        gp.wait_value = step + 1
        nxt = (step + 1 if self._fused_now else step) % _RING
        if tb.count:
            self._grid_update_launch(gp, tb.view(), par, self._status_ptr(nxt), _stream_ptr())
            self._slot_clean[nxt] = True
        else:
            # no blocks, nothing to update: still a party to the step barrier
            self._call("mpm_wait_step", C.byref(gp), self._gref(), _stream_ptr())
        self._vel_dt = self.dt

    def _after_gather(self, slot, step):
        if self._status_alias and self._guard_alias:
            self._call("mpm_status_publish", self._status_ptr(slot),
                       self._status_alias + slot * _capi.STATUS_BYTES, self._guard_word.data_ptr(),
                       self._guard_alias + 4 * slot, _stream_ptr())
        else:
            self._status_host[slot].copy_(self._status[slot], non_blocking=True)
            self._guard_host[slot:slot + 1].copy_(self._guard_word, non_blocking=True)
        self._status_events[slot].record()
        if self._defer:
            self._unconsumed = (slot, step)
        else:
            self._consume(slot, step)

    # -- collective (host-paced) step ---------------------------------------------------------
    def _check_wait_error(self):
        if int(self._mailbox[MB_WAIT_ERR].item()):
            raise BarrierTimeoutError(
                f"worker {self.wid}: a peer's step signal did not arrive within "
                f"{self.wait_timeout_ms} ms (device-side barrier of the grid update)")

    def _collective_step(self):
        """Drain, agree, reset the replicated guard, then one step with the host collectives of
        _post_barrier.  Returns True when some rank still needs a rebuild afterwards."""
        rt = self.runtime
        torch.cuda.current_stream().synchronize()     # none of my kernels / remote atomics in flight
        self._check_wait_error()
        rt.host_barrier()                             # ... nor anybody else's
        self._call("mpm_fill_i32", self._guard_word.data_ptr(), 1, _INT_MAX, _stream_ptr())
        # The step word too: with split transfers a fast rank may have signalled a step that a
        # slower peer's late guard then voided (its clear / P2G of step s + 1 ran and stored
        # s + 2 before the peer's G2P of step s raised the guard).  Left in place, that stale
        # value would satisfy the peers' wait of the RE-RUN step while this rank's new scatter is
        # still in flight.  Everything is drained here, so the word goes back to "steps below
        # _global_step are complete".
        self._call("mpm_fill_i32", self._mailbox.data_ptr() + 4 * MB_STEP, 1, self._global_step,
                   _stream_ptr())
        torch.cuda.current_stream().synchronize()
        rt.host_barrier()                             # every copy of the guard is reset
        step = self._global_step
        self._guard = self._make_guard(step)
        self._defer = False
        self._collective = True
        try:
            self.step_pre_barrier(step)
            self.step_post_barrier(step)
        finally:
            self._collective = False
            self._guard = None
        self.collective_steps += 1
        return bool(rt.all_gather_i64([int(self.flags.rebuild_needed)])[:, 0].any())

    def run_step(self, step):
        """One host-paced step (peer rows still read in place, barrier still on the device)."""
        if step != self._global_step:
            raise ContractViolationError(f"steps run in order: expected {self._global_step}, got {step}")
        with torch.cuda.device(self.device):
            self._collective_step()

    # -- device-paced frame ----------------------------------------------------------------------
    def _enqueue_guarded(self):
        step = self._global_step
        snap = self._snapshot()
        self._guard = self._make_guard(step)
        self._defer = True
        self._unconsumed = None
        try:
            self.step_pre_barrier(step)
            self.step_post_barrier(step)
        finally:
            self._defer = False
            self._guard = None
        cur = self._unconsumed
        if cur is None:
            # a rank without particles ran no gather: still record where the guard stood
            slot = step % _RING
            self._status_host[slot].zero_()
            self._guard_host[slot:slot + 1].copy_(self._guard_word, non_blocking=True)
            self._status_events[slot].record()
            cur = (slot, step)
        return cur[0], step, snap

    def _consume_peer(self, slot, step):
        self._status_events[slot].synchronize()
        g = int(self._guard_host[slot])
        if g < step:
            return SKIPPED          # the device skipped this step: some rank asked for a rebuild before it
        self._consume(slot, step)
        return RAISED if g == step else DONE

    def _peer_plan(self):
        """The single-worker step plan (worker.py) plus the peer fields of mpm_step_plan."""
        self.fuse_clear = False
        plan = self._step_plan()
        gp = self._grid_params()
        self._fill_peers(gp, plan=plan)
        C.memmove(C.byref(plan.grid), C.byref(gp), C.sizeof(_capi.GridParams))
        g = self._make_guard(0)
        plan.n_peer_words = g.n_peer_words
        for k in range(g.n_peer_words):
            plan.peer_guard_words[k] = g.peer_words[k]
        plan.signal_word = self._mailbox.data_ptr() + 4 * MB_STEP
        plan.guard_host = self._guard_host.data_ptr()
        plan.guard_word = self._guard_word.data_ptr()
        for k in range(2 * _capi.MAX_STATUS_RING):
            plan.time_events[k] = None
        return plan

    def _device_paced_batched(self, spf):
        """Steady-state steps enqueued from C (mpm_enqueue_steps), up to two batches in flight.
        Host bookkeeping advances when a step's status block is read.  Returns True when the
        next step must be collective (some rank asked for a rebuild)."""
        pending = []
        next_step = self._global_step
        enq = self._frame_steps
        while self._frame_steps < spf:
            while len(pending) <= self.batch_steps and enq < spf:
                n = min(self.batch_steps, spf - enq)
                plan = self._peer_plan()
                plan.transfer.dt_gather = float(self._vel_dt if not pending else self.dt)
                self.kernel_calls += 1
                _capi.check(self.lib.mpm_enqueue_steps(C.byref(plan), next_step, n, _stream_ptr()),
                            "mpm_enqueue_steps")
                pending += list(range(next_step, next_step + n))
                next_step += n
                enq += n
            step = pending.pop(0)
            slot = step % _RING
            self._slot_clean[slot] = False
            outcome = self._consume_peer(slot, step)
            if outcome == SKIPPED:
                self.speculative_discards += 1 + len(pending)
                return True
            # step `step` ran to completion on every rank
            self._global_step = step + 1
            self._vel_dt = self.dt
            self.flags.steps_since_rebuild += 1
            self._frame_steps += 1
            self.device_paced_steps += 1
            self.batched_steps += 1
            self.frame_dts.append(self.dt)
            if outcome == RAISED or self.flags.rebuild_needed:
                self.speculative_discards += len(pending)
                return True
        return False

    def run_frame(self):
        self.begin_frame()
        spf = self.params.steps_per_frame
        with torch.cuda.device(self.device):
            if self.cfl_mode:
                self._run_frame_collective_cfl()
            else:
                self.dt = self.params.dt
                inflight = []
                # The first step of a frame is collective (agree on rebuilds the frame-end flush may
                # have asked for) -- unless lazy_flush left the gather pending and nothing read the
                # store since: then the frame boundary is invisible to the device-paced pipeline.
                # Store reads (which flush) must be SPMD: every rank or none.
                collective = self._need_collective or not (self.lazy_flush and self._pending_gather)
                while self._frame_steps < spf:
                    if collective:
                        collective = self._collective_step()
                        self._frame_steps += 1
                        self.frame_dts.append(self.dt)
                        continue
                    if not inflight and self.batch_steps > 0 and self._can_batch():
                        collective = self._device_paced_batched(spf)
                        continue
                    if self._frame_steps + len(inflight) < spf and len(inflight) < self.depth \
                            and not (inflight and self.batch_steps > 0 and self._can_batch()):
                        inflight.append(self._enqueue_guarded())
                        continue
                    slot, step, snap = inflight.pop(0)
                    outcome = self._consume_peer(slot, step)
                    if outcome == SKIPPED:
                        self._restore(snap)
                        self.speculative_discards += 1 + len(inflight)
                        inflight, collective = [], True
                        continue
                    self._frame_steps += 1
                    self.device_paced_steps += 1
                    self.frame_dts.append(self.dt)
                    if outcome == RAISED or self.flags.rebuild_needed:
                        if inflight:
                            self._restore(inflight[0][2])
                            self.speculative_discards += len(inflight)
                        inflight, collective = [], True
            self._need_collective = collective
            if self._pending_gather and not self.lazy_flush:
                self._flush_gather()

    def _run_frame_collective_cfl(self):
        from .domain import cfl_dt
        c_sound = self.global_sound_speed()
        t = 0.0
        while t < self.params.frame_dt - 1e-12:
            vmax = self.runtime.global_vmax((self._global_step - 2) % 3)
            self.dt = cfl_dt(vmax + c_sound, self.params, self.params.frame_dt - t)
            self._collective_step()
            t += self.dt
            self._frame_steps += 1
            self.frame_dts.append(self.dt)
