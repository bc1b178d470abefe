"""CudaWorker: the reference's `Worker` surface over the B200 CUDA core.

Mirrors /root/reference/pkg/src/mpmbench/pipeline.py:788-1238 (Worker), with
ParticleStore (particles.py:268-487), BlockTable (grid.py:325-401) and GridStore
(grid.py:415-454) re-hosted on device buffers.  Every phase is one call through the C ABI
(include/mpm_b200.h); this module only sequences them, owns the buffers (4x growth rule) and
maps counters / status codes onto the reference's exceptions.  There is no CPU path: without
libmpm_b200.so or a CUDA device, construction raises ResourceError.

Host/device protocol of one substep (pipeline.py:905-940):
    [rebuild | clear(par)] -> [g2p2g | p2g] -> barrier -> grid update (+ peer rows) -> [g2p]
    -> 56-byte status block D2H (free-zone flag, max speed^2, counters) -> host decides
       whether the next step rebuilds (pipeline.py:1102-1104).
"""
from __future__ import annotations

import ctypes as C
import logging
import math
import os
import time

import numpy as np
import torch

from . import _capi
from ._capi import StepStatus, StoreView, TableView, TransferParams, check
from .domain import Material, MaterialKind, SimParams, cfl_dt
from .errors import (ConfigError, ContractViolationError, ModeConflictError, RejectedInputError,
                     SpatialDomainError)
from .memory import DeviceBuffer
from .options import (C_ADDRESS_ERR, FREE_ZONE_HI_CELLS, FREE_ZONE_LO_CELLS, FUSED_MARGIN_CELLS,
                      N_COUNTERS, BoundaryBox, PipelineOptions, StepFlags)

log = logging.getLogger(__name__)

CELL_BIAS = 64
CH_POS, CH_VEL, CH_C, CH_MASS, CH_DEF, CH_PLASTIC = 0, 3, 6, 15, 16, 25
LW = 32
_INT_MAX = 0x7FFFFFFF
_PHASES = ("rebuild", "sort", "p2g", "grid", "g2p")
_RING = 16          # status slots: two batches of speculative steps in flight
_BATCH = 4          # steps enqueued per C call in steady state


def channels_for(kind: int) -> int:
    """particles.py:24-31: 17 channels for the fluid (J), 25 for F; +1 plastic scalar."""
    kind = int(kind)
    if kind == MaterialKind.WEAKLY_COMPRESSIBLE_FLUID:
        return 17
    if kind == MaterialKind.FIXED_COROTATED:
        return 25
    return 26


def _pow2_at_least(n: int) -> int:
    return 1 << max(int(n) - 1, 1).bit_length()


# --------------------------------------------------------------------------------------
# particle store (particles.py:268-487)
# --------------------------------------------------------------------------------------
class CudaParticleStore:
    """AoSoA particle storage on the device: data[group][channel][32] fp32, double-buffered
    so a rebuild permutes from the old copy into the new one."""

    def __init__(self, kind, lane_width, device):
        if int(lane_width) != LW:
            raise ConfigError(f"the CUDA core maps one warp to one lane group: lane_width must be {LW}")
        self.kind = int(kind)
        self.lane_width = LW
        self.nch = channels_for(kind)
        self.device = device
        mk = lambda dt, shape=(): [DeviceBuffer(dt, shape, device), DeviceBuffer(dt, shape, device)]
        self._data = mk(torch.float32, (self.nch, LW))
        self._orig_id = mk(torch.int64, (LW,))
        self._lane_meta = mk(torch.int16, (LW,))
        self._group_len = mk(torch.int32)
        self._group_block = mk(torch.int32)
        self._group_start = mk(torch.int32)
        self._group_ctx = mk(torch.int32, (LW,))
        self.cur = 0
        self.n_groups = 0
        self.count = 0
        self._staged = []
        self.staged_count = 0
        self._next_id = 0
        self._pin = {}
        self.has_sink = False   # set by the worker: sunk lanes (orig_id -1) are skipped by readbacks
        self._table = None   # set by the worker: group_origin comes from the block table
        self._before_read = None   # set by the worker: completes a lazily pending gather

    # -- views for the C ABI --
    def view(self, which=None) -> StoreView:
        k = self.cur if which is None else which
        return StoreView(self._data[k].ptr, self._orig_id[k].ptr, self._lane_meta[k].ptr,
                         self._group_len[k].ptr, self._group_block[k].ptr,
                         self._group_start[k].ptr, self.n_groups if k == self.cur else 0, self.nch,
                         self._group_ctx[k].ptr)

    @property
    def realloc_count(self) -> int:
        return sum(b.realloc_count for pair in (self._data, self._orig_id, self._lane_meta,
                                                self._group_len, self._group_block,
                                                self._group_start, self._group_ctx) for b in pair)

    # -- population (particles.py:309-334) --
    def default_deformation(self, n):
        if self.kind == MaterialKind.WEAKLY_COMPRESSIBLE_FLUID:
            return np.ones((n, 1), dtype=np.float32)
        return np.tile(np.eye(3, dtype=np.float32).reshape(9), (n, 1))

    def stage_append(self, positions, velocities, masses, deformation=None, affine=None, ids=None):
        """Queue host particles for the next rebuild (particles.py:309-334).  Arrays are kept
        compact (x, v, m [, F|J, C]); the channel rows are laid out on the device.  Pinned
        float32 / int64 torch tensors are uploaded as they are (no staging copy)."""
        if isinstance(positions, torch.Tensor) and deformation is None and affine is None:
            tp, tv = positions, velocities
            n = tp.shape[0]
            if n == 0:
                return 0
            if tp.ndim != 2 or tp.shape[1] != 3 or tuple(tv.shape) != tuple(tp.shape):
                raise RejectedInputError(f"positions / velocities must have shape (n, 3), got "
                                         f"{tuple(tp.shape)} / {tuple(tv.shape)}")
            tp = tp.to(torch.float32).contiguous()
            tv = tv.to(torch.float32).contiguous()
            tm = masses if isinstance(masses, torch.Tensor) else np.asarray(masses, dtype=np.float32)
            if ids is None:
                ti = torch.arange(self._next_id, self._next_id + n, dtype=torch.int64)
                self._next_id += n
            else:
                ti = torch.as_tensor(ids, dtype=torch.int64).contiguous()
                self._next_id = max(self._next_id, int(ti.max()) + 1)
            self._staged.append((tp, tv, tm, None, None, ti))
            self.staged_count += n
            return n
        pos = np.atleast_2d(np.asarray(positions))
        n = pos.shape[0]
        if n == 0:
            return 0
        if pos.shape[1] != 3:
            raise RejectedInputError(f"positions must have shape (n, 3), got {pos.shape}")
        vel = np.atleast_2d(np.asarray(velocities))
        if vel.shape != pos.shape:
            raise RejectedInputError(f"velocities must have shape {pos.shape}, got {vel.shape}")
        pos = np.ascontiguousarray(pos, dtype=np.float32)
        vel = np.ascontiguousarray(vel, dtype=np.float32)
        mass = np.asarray(masses, dtype=np.float32)
        if mass.ndim:
            mass = np.ascontiguousarray(np.broadcast_to(mass, (n,)))
        defo = None if deformation is None else \
            np.ascontiguousarray(np.asarray(deformation, dtype=np.float32).reshape(n, -1))
        aff = None if affine is None else \
            np.ascontiguousarray(np.asarray(affine, dtype=np.float32).reshape(n, 9))
        if ids is None:
            ids = np.arange(self._next_id, self._next_id + n, dtype=np.int64)
            self._next_id += n
        else:
            ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64).reshape(n))
            self._next_id = max(self._next_id, int(ids.max()) + 1)
        self._staged.append((pos, vel, mass, defo, aff, ids))
        self.staged_count += n
        return n

    def _default_state(self, flat):
        """F = I (J = 1), C = 0, plastic scalar at rest (particles.py:309-320)."""
        flat[:, CH_DEF] = 1.0
        if self.kind != MaterialKind.WEAKLY_COMPRESSIBLE_FLUID:
            flat[:, CH_DEF + 4] = 1.0
            flat[:, CH_DEF + 8] = 1.0
        if self.nch > CH_PLASTIC:
            flat[:, CH_PLASTIC] = 1.0 if self.kind == MaterialKind.SNOW else 0.0

    def _pinned(self, tag, shape, dtype):
        """Grow-only pinned host staging buffers (reused across uploads / readbacks)."""
        need = int(np.prod(shape))
        buf = self._pin.get(tag)
        if buf is None or buf.numel() < need or buf.dtype != dtype:
            buf = self._pin[tag] = torch.empty(max(need, 1), dtype=dtype).pin_memory()
        return buf[:need].view(*shape)

    def take_staged(self):
        """Upload the staged particles: pinned host buffers -> device, then the flat channel rows
        [n, nch] (fp32) and ids [n] that the rebuild kernels read."""
        if not self._staged:
            return None, None, 0
        n = self.staged_count
        dev = self.device
        if all(isinstance(e[0], torch.Tensor) for e in self._staged):
            # tensors (ideally pinned): straight H2D copies into the flat rows
            # the rows are laid out by one kernel per staged batch (mpm_stage_particles)
            flat = torch.empty((n, self.nch), dtype=torch.float32, device=dev)
            dids = torch.empty(n, dtype=torch.int64, device=dev)
            lib, stream = _capi.lib(), _stream_ptr()
            o = 0
            for tp, tv, tm, _, _, ti in self._staged:
                k = tp.shape[0]
                dpos, dvel = tp.to(dev, non_blocking=True), tv.to(dev, non_blocking=True)
                dmass, scalar = None, 0.0
                if isinstance(tm, torch.Tensor):
                    dmass = tm.to(dev, torch.float32, non_blocking=True).contiguous()
                elif tm.ndim:
                    dmass = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(tm, (k,)))).to(dev)
                else:
                    scalar = float(tm)
                check(lib.mpm_stage_particles(dpos.data_ptr(), dvel.data_ptr(),
                                              dmass.data_ptr() if dmass is not None else None, scalar, k,
                                              self.nch, self.kind, flat.data_ptr() + 4 * o * self.nch, stream),
                      "mpm_stage_particles")
                dids[o:o + k] = ti.to(dev, non_blocking=True)
                o += k
            self._staged.clear()
            self.staged_count = 0
            return flat, dids, n
        self._staged = [tuple(x.numpy() if isinstance(x, torch.Tensor) else x for x in e)
                        for e in self._staged]
        hpos = self._pinned("pos", (n, 3), torch.float32)
        hvel = self._pinned("vel", (n, 3), torch.float32)
        hids = self._pinned("ids", (n,), torch.int64)
        hmass = self._pinned("mass", (n,), torch.float32)
        o = 0
        extras = []
        for pos, vel, mass, defo, aff, ids in self._staged:
            k = len(ids)
            hpos[o:o + k].copy_(torch.from_numpy(pos))
            hvel[o:o + k].copy_(torch.from_numpy(vel))
            hids[o:o + k].copy_(torch.from_numpy(ids))
            if mass.ndim:
                hmass[o:o + k].copy_(torch.from_numpy(np.ascontiguousarray(mass).copy() if not mass.flags.writeable else mass))
            else:
                hmass[o:o + k].fill_(float(mass))
            if defo is not None or aff is not None:
                extras.append((o, k, defo, aff))
            o += k
        self._staged.clear()
        self.staged_count = 0
        flat = torch.zeros((n, self.nch), dtype=torch.float32, device=dev)
        flat[:, CH_POS:CH_POS + 3] = hpos.to(dev, non_blocking=True)
        flat[:, CH_VEL:CH_VEL + 3] = hvel.to(dev, non_blocking=True)
        flat[:, CH_MASS] = hmass.to(dev, non_blocking=True)
        self._default_state(flat)
        for o, k, defo, aff in extras:
            if defo is not None:
                flat[o:o + k, CH_DEF:CH_DEF + defo.shape[1]] = torch.from_numpy(defo).to(dev)
            if aff is not None:
                flat[o:o + k, CH_C:CH_C + 9] = torch.from_numpy(aff).to(dev)
        dids = hids.to(dev, non_blocking=True)
        return flat, dids, n

    # -- readback (lazy D2H views in the reference's layout / dtype) --
    def _g(self, bufs):
        if self._before_read is not None:
            self._before_read()
        return bufs[self.cur].data[:self.n_groups]

    @property
    def data(self):
        return self._g(self._data).to(torch.float64).cpu().numpy()

    def set_data(self, array):
        """Upload particle channels given in the reference layout [n_groups, nch, 32] (the
        reference's tests write into `store.data` in place, e.g. fault injection)."""
        a = torch.as_tensor(np.ascontiguousarray(array, dtype=np.float32), device=self.device)
        self._g(self._data).copy_(a)

    @property
    def orig_id(self):
        return self._g(self._orig_id).cpu().numpy()

    @property
    def lane_key(self):
        return (self._g(self._lane_meta).cpu().numpy().view(np.uint16) & 0x3FF).astype(np.int64)

    @property
    def quarantined(self):
        return ((self._g(self._lane_meta).cpu().numpy().view(np.uint16) >> 15) & 1).astype(np.uint8)

    @property
    def group_len(self):
        return self._g(self._group_len).cpu().numpy()

    @property
    def group_block(self):
        return self._g(self._group_block).cpu().numpy()

    @property
    def group_origin(self):
        origin = self._table._origin.data[:self._table.count, :3].cpu().numpy()
        return origin[self.group_block.astype(np.int64)].astype(np.int32)

    def state_with_ids(self):
        """All stored lanes (quarantined included) in (group, lane) order: flat f64 [n, nch], ids."""
        if self._before_read is not None:
            self._before_read()
        n = self.count
        flat = torch.zeros((max(n, 1), self.nch), dtype=torch.float32, device=self.device)
        ids = torch.zeros(max(n, 1), dtype=torch.int64, device=self.device)
        if n:
            v = self.view()
            check(_capi.lib().mpm_gather_state(C.byref(v), flat.data_ptr(), ids.data_ptr(),
                                               _stream_ptr()), "mpm_gather_state")
        flat, ids = flat[:n].to(torch.float64).cpu().numpy(), ids[:n].cpu().numpy()
        if self.has_sink:
            keep = ids >= 0
            flat, ids = flat[keep], ids[keep]
        return flat, ids

    def positions_with_ids(self, dtype=np.float64):
        """particles.py:466-475: positions of every stored particle (quarantined included) and
        their ids, in (group, lane) order."""
        if self._before_read is not None:
            self._before_read()
        n = self.count
        if not n:
            return np.zeros((0, 3), dtype=dtype), np.zeros(0, dtype=np.int64)
        pos = torch.empty((n, 3), dtype=torch.float32, device=self.device)
        ids = torch.empty(n, dtype=torch.int64, device=self.device)
        v = self.view()
        check(_capi.lib().mpm_gather_positions(C.byref(v), pos.data_ptr(), ids.data_ptr(),
                                               _stream_ptr()), "mpm_gather_positions")
        hpos = self._pinned("out_pos", (n, 3), torch.float32)
        hids = self._pinned("out_ids", (n,), torch.int64)
        hpos.copy_(pos, non_blocking=True)
        hids.copy_(ids, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if self.has_sink:
            keep = hids.numpy() >= 0
            return hpos.numpy()[keep].astype(dtype or np.float32), hids.numpy()[keep]
        if dtype is None:
            # zero-copy views of the pinned readback buffers, valid until the next readback
            return hpos.numpy(), hids.numpy()
        return hpos.numpy().astype(dtype), hids.numpy().copy()

    def positions_with_ids_async(self):
        """positions_with_ids(dtype=None) without the host wait: the snapshot is gathered on the
        compute stream into one of two device buffers and copied to pinned host memory on a copy
        stream, so the transfer overlaps whatever the caller enqueues next (the upload and the
        first substeps of the following frame).  Returns a PendingReadback; .wait() gives the
        (positions float32 [n, 3], ids int64 [n]) views, valid until the second next call."""
        if self._before_read is not None:
            self._before_read()
        n = self.count
        k = self._rb_parity = 1 - getattr(self, "_rb_parity", 1)
        if not hasattr(self, "_rb_stream"):
            self._rb_stream = torch.cuda.Stream(device=self.device)
            self._rb_done = [None, None]
            self._rb_dev = [None, None]
        main = torch.cuda.current_stream()
        if self._rb_done[k] is not None:
            main.wait_event(self._rb_done[k])      # the copy that last used these buffers
        dev = self._rb_dev[k]
        if dev is None or dev[0].shape[0] < n:
            dev = self._rb_dev[k] = (torch.empty((max(n, 1), 3), dtype=torch.float32, device=self.device),
                                     torch.empty(max(n, 1), dtype=torch.int64, device=self.device))
        hpos = self._pinned(f"out_pos{k}", (n, 3), torch.float32)
        hids = self._pinned(f"out_ids{k}", (n,), torch.int64)
        if n:
            v = self.view()
            check(_capi.lib().mpm_gather_positions(C.byref(v), dev[0].data_ptr(), dev[1].data_ptr(),
                                                   _stream_ptr()), "mpm_gather_positions")
            gathered = torch.cuda.Event()
            gathered.record(main)
            self._rb_stream.wait_event(gathered)
            with torch.cuda.stream(self._rb_stream):
                hpos.copy_(dev[0][:n], non_blocking=True)
                hids.copy_(dev[1][:n], non_blocking=True)
        done = self._rb_done[k] = torch.cuda.Event()
        done.record(self._rb_stream)
        return PendingReadback(done, hpos, hids)

    def _aggregates(self):
        if self._before_read is not None:
            self._before_read()
        out = torch.zeros(5, dtype=torch.float64, device=self.device)
        v = self.view()
        check(_capi.lib().mpm_particle_aggregates(C.byref(v), out.data_ptr(), _stream_ptr()),
              "mpm_particle_aggregates")
        return out.cpu().numpy()

    def total_mass(self) -> float:
        return float(self._aggregates()[0])

    def total_momentum(self):
        return self._aggregates()[1:4].copy()

    def kinetic_energy(self) -> float:
        return float(self._aggregates()[4])


class _Ms:
    """A kernel duration already read from its CUDA events.  The events of batched steps are a
    small ring that later batches record again, so their elapsed time is taken when the step is
    consumed; `kernel_events` entries keep the (name, a, b) shape with a.elapsed_time(b)."""
    __slots__ = ("ms", "age")

    def __init__(self, ms, age=-1):
        self.ms = float(ms)
        self.age = int(age)       # steps since the last rebuild when the kernel ran

    def elapsed_time(self, _other=None):
        return self.ms


class PendingReadback:
    """A snapshot on its way to pinned host memory (CudaParticleStore.positions_with_ids_async)."""

    def __init__(self, done, hpos, hids):
        self._done, self._hpos, self._hids = done, hpos, hids

    def wait(self):
        self._done.synchronize()
        return self._hpos.numpy(), self._hids.numpy()


# --------------------------------------------------------------------------------------
# block table (grid.py:325-401) and nodal buffers (grid.py:415-454)
# --------------------------------------------------------------------------------------
class CudaBlockTable:
    def __init__(self, device):
        self.device = device
        self._codes = DeviceBuffer(torch.int64, (), device)
        self._origin = DeviceBuffer(torch.int32, (4,), device)
        self._neighbor = DeviceBuffer(torch.int32, (27,), device)
        self._touched = [DeviceBuffer(torch.uint8, (), device), DeviceBuffer(torch.uint8, (), device)]
        self._hkeys = DeviceBuffer(torch.int64, (), device)
        self._hvals = DeviceBuffer(torch.int32, (), device)
        self._hfirst = DeviceBuffer(torch.int32, (), device)
        self.hash_cap = 0
        self.count = 0
        self.n_gblocks = 0

    @property
    def realloc_count(self) -> int:
        return sum(b.realloc_count for b in (self._codes, self._origin, self._neighbor,
                                             self._touched[0], self._touched[1], self._hkeys,
                                             self._hvals, self._hfirst))

    def ensure_hash(self, cap: int):
        for b in (self._hkeys, self._hvals, self._hfirst):
            if b.capacity < cap:
                b.capacity = 0          # exact power-of-two sizing, contents are rebuilt anyway
                b.len = 0
                b.data = torch.empty(cap, dtype=b.dtype, device=self.device)
                b.capacity = cap
                b.realloc_count += 1
                DeviceBuffer.generation += 1
        self.hash_cap = cap

    def view(self) -> TableView:
        t = TableView()
        t.codes, t.origin, t.neighbor = self._codes.ptr, self._origin.ptr, self._neighbor.ptr
        t.touched[0], t.touched[1] = self._touched[0].ptr, self._touched[1].ptr
        t.count, t.n_gblocks = self.count, self.n_gblocks
        return t

    @property
    def codes(self):
        return self._codes.data[:self.count].cpu().numpy()

    @property
    def neighbor(self):
        return self._neighbor.data[:self.n_gblocks].cpu().numpy()

    @property
    def touched(self):
        return [self._touched[k].data[:self.count].cpu().numpy() for k in (0, 1)]

    def touched_indices(self, buffer: int = 0):
        return np.flatnonzero(self.touched[buffer])


class CudaGrid:
    """raw[0], raw[1], vel (+ vel_old): float4 nodes [pblock][64] on the device.  The numpy
    properties return the reference's channel-major float64 layout [pblock, 4, 64]."""

    def __init__(self, device, deterministic=False):
        self.device = device
        # deterministic mode: a raw node is four int64 (rint(c 2^40), rint(c 2^32) x3), pipeline.py:43-44
        rdt = torch.int64 if deterministic else torch.float32
        self.deterministic = bool(deterministic)
        self._raw = [DeviceBuffer(rdt, (64, 4), device), DeviceBuffer(rdt, (64, 4), device)]
        self._vel = DeviceBuffer(torch.float32, (64, 4), device)
        self._vel_old = None
        self.count = 0

    @property
    def realloc_count(self) -> int:
        n = self._raw[0].realloc_count + self._raw[1].realloc_count + self._vel.realloc_count
        return n + (self._vel_old.realloc_count if self._vel_old is not None else 0)

    def _ref_layout(self, buf):
        return buf.data[:self.count].to(torch.float64).permute(0, 2, 1).contiguous().cpu().numpy()

    @property
    def raw(self):
        return [self._ref_layout(self._raw[0]), self._ref_layout(self._raw[1])]

    @property
    def vel(self):
        return self._ref_layout(self._vel)

    def set_vel(self, array):
        """Upload nodal velocities given in the reference layout [count, 4, 64] (painted-grid
        tests, tests/test_pipeline.py:28-37 of the reference)."""
        a = torch.as_tensor(np.ascontiguousarray(array, dtype=np.float32), device=self.device)
        self._vel.data[:self.count].copy_(a.permute(0, 2, 1))

    @property
    def vel_old(self):
        if self._vel_old is None:
            return None
        return self._ref_layout(self._vel_old)[:, 1:4, :]


def _stream_ptr() -> int:
    """cudaStream_t of the current torch stream.  torch.cuda.current_stream() builds a Stream
    object through several Python layers (~15 us, a third of the host time of a 64 K-particle
    frame); the raw getter is one C call."""
    try:
        return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
    except AttributeError:              # a torch without the raw getter
        return torch.cuda.current_stream().cuda_stream


# --------------------------------------------------------------------------------------
# worker (pipeline.py:788-1238)
# --------------------------------------------------------------------------------------
class CudaWorker:
    """Drop-in for `mpmbench.pipeline.Worker` on one CUDA device."""

    def __init__(self, wid, runtime, params: SimParams, material: Material,
                 boundary: BoundaryBox | None, options: PipelineOptions | None = None,
                 device=None, count_stats: bool = True, fuse_clear: bool = False,
                 lazy_flush: bool = False):
        _capi.require_device()
        self.lib = _capi.lib()
        self.device = torch.device(device if device is not None else "cuda:0")
        self.wid = wid
        self.runtime = runtime
        self.params = params
        self.material = material
        self.boundary = boundary
        self.options = options if options is not None else PipelineOptions()
        if self.options.fusion != "merged" or self.options.sort == "full_every_step":
            raise ConfigError("the CUDA core implements fusion=merged and sort=amortized|none_between "
                              "(the other arms re-measure CPU ablations, SURVEY.md section 2 row 13)")
        if self.options.deterministic and int(material.kind) not in (0, 1):
            raise ConfigError("deterministic fixed-point accumulation covers the reference's material "
                              "kinds (fluid, fixed-corotated)")
        with torch.cuda.device(self.device):
            self.store = CudaParticleStore(material.kind, params.lane_width, self.device)
            self.table = CudaBlockTable(self.device)
            self.grid = CudaGrid(self.device, self.options.deterministic)
            self.store._table = self.table
            # status ring: one block per in-flight step (zone flag, max speed^2, counters); the
            # counters of a slot accumulate over every step that used it
            self._status = torch.zeros((_RING, _capi.STATUS_BYTES // 8), dtype=torch.int64,
                                       device=self.device)
            self._status_host = torch.zeros((_RING, _capi.STATUS_BYTES // 8),
                                            dtype=torch.int64).pin_memory()
            # device alias of the host ring: status blocks are stored to it by kernels
            # (mpm_status_publish / the grid update), not copied -- a kernel -> copy -> kernel chain
            # idles the device for a copy-engine round trip per step
            self._status_alias = self.lib.mpm_host_alias(self._status_host.data_ptr())
            self._status_views = None
            self._status_events = [torch.cuda.Event() for _ in range(_RING)]
            self._time_events = [torch.cuda.Event(enable_timing=True) for _ in range(2 * _BATCH * 2)]
            for ev in self._status_events + self._time_events:
                ev.record()          # events are created lazily: force the handles into existence
            self._slot_clean = [True] * _RING
            self._guard_word = torch.full((1,), _INT_MAX, dtype=torch.int32, device=self.device)
            self._scalars = torch.zeros(16, dtype=torch.int32, device=self.device)
            self._scalars_host = torch.zeros(16, dtype=torch.int32).pin_memory()
            self._rebuild_event = torch.cuda.Event()
            self._rebuild_event.record()
            # group count of either half of the particle store, kept on the device by the rebuild
            # that filled it (mpm_rebuild_plan.n_groups_out): the next rebuild reads it there
            self._ngroups_dev = torch.zeros(2, dtype=torch.int32, device=self.device)
            self._ngroups_dev_valid = [False, False]
            # step clock of CFL-auto frames (mpm_step_clock: dt[2], t, reserved), device-resident
            self._clock = torch.zeros(4, dtype=torch.float64, device=self.device)
            self._clock_host = torch.zeros(4, dtype=torch.float64).pin_memory()
        self.flags = StepFlags(deterministic_mode=bool(self.options.deterministic))
        self._node_bytes = 32 if self.options.deterministic else 16
        self.conservation = []
        self.rebuild_steps = []
        self.dt = params.dt
        self._vel_dt = params.dt
        self._global_step = 0
        self._pending_gather = False
        self._flushing = False
        self._pending_full_clear_parity = -1
        self._published_codes = (None, 0)
        self._peer_map = [None] * runtime.n_workers
        self._peer_states = None
        self._fused_now = False
        self._fused_fallback_logged = False
        self._phase_ms = {k: 0.0 for k in _PHASES}
        self._frame_steps = 0
        self._frame_rebuilds = 0
        self.cfl_mode = False
        # CFL-auto frames paced by the device (mpm_step_clock): the grid update computes the next
        # step size from the max speed of two steps earlier and ends the frame itself, so adaptive
        # frames are enqueued ahead like fixed-dt ones.  False = the host computes dt every step.
        self.device_clock = True
        self._use_clock = False       # set for the duration of a device-clocked frame
        self._clock_valid = False     # the device clock holds dt of step _global_step, t = 0
        self._flushing_gather = False
        self._last_dt = 0.0
        self._last_frame_end = False
        self._removed_seen = [0] * _RING
        self._sunk_pending = False
        self.frame_dts = []
        self.count_stats = bool(count_stats)
        self.fuse_clear = bool(fuse_clear)
        # lazy_flush: a frame may end with the fused transfer's gather still pending (the reference
        # flushes it at every frame end, pipeline.py:877-880, because its harness reads positions
        # there).  The flush then happens on the first access to the particle store, so what a
        # caller observes is unchanged, and back-to-back frames stay fused across the boundary.
        self.lazy_flush = bool(lazy_flush)
        self.store._before_read = self._ensure_flushed
        self.last_perm = None
        self.last_gidx = None
        self._scratch = {}
        self._scratch_allocs = 0
        self.kernel_calls = 0
        self._tail_done = False
        self._tail_g2p_done = False
        # Opt-in: replay the rebuild kernels as a CUDA graph once the scene is in steady state (same
        # particle count, no buffer moved for four rebuilds).  Measured (profiles/experiments/README.md):
        # the host's part of a rebuild at 64 K particles falls from ~130 to ~40 us, the frame by 0-7 %;
        # nothing at 171 K and above (the chain is device-bound there), and a scene whose count keeps
        # changing (fountain: emitter + sink) pays for captures it never reuses.  Off by default.
        self.rebuild_graph = os.environ.get("MPM_REBUILD_GRAPH", "0") == "1"
        self.rebuild_graph_max = 200_000   # ... up to this many particles
        self.rebuild_graph_replays = 0
        self._rb_cache = {}           # store half -> (key, plan, result) of the last rebuild out of it
        self._rb_shape, self._rb_stable = None, 0
        self._rebuild_next_n = 0
        self._rebuild_next = 0        # steps mpm_rebuild may enqueue behind the rebuild step (frame drivers)
        self._rebuild_enqueued = 0    # ... and how many it did
        self._tp_gather, self._tp_scatter, self._gp_tail = TransferParams(), TransferParams(), _capi.GridParams()
        self._time_rot = 0
        self.time_kernels = False     # bench: CUDA events around the step kernels
        self.profile_all_phases = False   # harness CSV: every gather is issued (and timed) from Python
        self.pipelined = True         # run_frame enqueues step s+1 before reading step s's flag
        self.batch_steps = _BATCH     # fixed-dt frames: steps per mpm_enqueue_steps call (0 = off)
        self._plan = None
        self._plan_stale = True
        self._guard_reset_in_rebuild = False
        self.speculative_discards = 0
        self.kernel_events = []
        self._frame_event_start = 0
        self._gp = None
        self._guard = None            # ctypes Guard of the step being enqueued (pipelined frames)
        self._defer = False           # leave gather statuses unread (pipelined frames)
        self._unconsumed = None
        m = material
        self._tp = TransferParams(
            mat_kind=int(m.kind), nch=self.store.nch, mu=float(m.mu), lam=float(m.lam),
            kappa=float(m.bulk_modulus), gamma=float(m.gamma),
            clamp_tension=int(bool(m.clamp_tension)), count_stats=int(self.count_stats),
            deterministic=int(bool(self.options.deterministic)),
            density=float(m.density), dx=float(params.dx), dt=float(params.dt),
            dt_gather=float(params.dt), flip_blend=float(params.flip_blend),
            margin_lo=FREE_ZONE_LO_CELLS, margin_hi=FREE_ZONE_HI_CELLS - 4.0,
            theta_c=float(m.theta_c), theta_s=float(m.theta_s), hardening=float(m.hardening),
            sand_alpha=math.sqrt(2.0 / 3.0) * 2.0 * math.sin(math.radians(m.friction_angle))
            / (3.0 - math.sin(math.radians(m.friction_angle))))

    # -- small helpers ----------------------------------------------------------------
    _TIMED = ("mpm_p2g", "mpm_g2p", "mpm_g2p2g", "mpm_grid_update", "mpm_clear")

    def _call(self, name, *args):
        self.kernel_calls += 1
        if self.time_kernels and name in self._TIMED:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            check(getattr(self.lib, name)(*args), name)
            b.record()
            self.kernel_events.append((name, a, b))
            return
        check(getattr(self.lib, name)(*args), name)

    def _scratch_i32(self, tag, n):
        """Tagged scratch (memory.py:72-114 ScratchPool): reused across rebuilds, 4x growth."""
        buf = self._scratch.get(tag)
        if buf is None:
            buf = self._scratch[tag] = DeviceBuffer(torch.int32, (), self.device)
        before = buf.realloc_count
        buf.ensure_capacity(max(int(n), 1), keep=False)
        self._scratch_allocs += buf.realloc_count - before
        return buf

    def _scratch_i64(self, tag, n):
        buf = self._scratch.get(tag)
        if buf is None:
            buf = self._scratch[tag] = DeviceBuffer(torch.int64, (), self.device)
        before = buf.realloc_count
        buf.ensure_capacity(max(int(n), 1), keep=False)
        self._scratch_allocs += buf.realloc_count - before
        return buf

    @property
    def counters(self):
        host = self._status.cpu().numpy()
        return host[:, 1:1 + N_COUNTERS].sum(axis=0).astype(np.int64)

    @property
    def frame_steps(self):
        return self._frame_steps

    @property
    def frame_rebuilds(self):
        return self._frame_rebuilds

    @property
    def phase_ms(self):
        """Per-frame phase times in the reference's five columns (pipeline.py:785).  rebuild / sort
        are host-timed (the rebuild synchronises anyway); the kernel phases come from CUDA events
        when `time_kernels` is on, the fused kernel split 50/50 (pipeline.py:1137-1138)."""
        out = dict(self._phase_ms)
        if self.time_kernels and self.kernel_events:
            torch.cuda.synchronize(self.device)
            for name, a, b in self.kernel_events[self._frame_event_start:]:
                ms = a.elapsed_time(b)
                if name == "mpm_p2g":
                    out["p2g"] += ms
                elif name == "mpm_g2p":
                    out["g2p"] += ms
                elif name == "mpm_g2p2g":
                    out["p2g"] += 0.5 * ms
                    out["g2p"] += 0.5 * ms
                else:
                    out["grid"] += ms
        return out

    @property
    def realloc_count(self):
        return (self.store.realloc_count + self.table.realloc_count + self.grid.realloc_count +
                self._scratch_allocs)

    # -- population (pipeline.py:831-850) -----------------------------------------------
    def seed_particles(self, positions, velocities, masses, ids):
        n = self.store.stage_append(positions, velocities, masses, ids=ids)
        self.flags.rebuild_needed = True
        return n

    def append_particles(self, positions, velocities, masses, ids=None):
        if len(np.atleast_2d(positions)) == 0:
            return 0
        if self.flags.fused_mode:
            raise ModeConflictError("cannot add particles while the fused G2P2G transfer is active")
        n = self.store.stage_append(positions, velocities, masses, ids=ids)
        if n:
            self.flags.rebuild_needed = True
        return n

    def replace_particles(self, positions, velocities, masses, ids):
        """Drop the current population and stage a new one from host arrays (the end-to-end
        entry of bench.py: same effect as a fresh worker + seed_particles, buffers reused)."""
        if self._pending_gather:
            self._pending_gather = False
        self.store.n_groups = 0
        self.store.count = 0
        self.flags.fused_mode = False
        return self.seed_particles(positions, velocities, masses, ids)

    # -- particle sink (not in the reference) -----------------------------------
    def set_sink(self, min_corner, max_corner):
        """Particles whose advected position lies in the box [min_corner, max_corner) leave the
        simulation: the gather that moved them there zeroes their mass and flags the lane, they stop
        scattering at once and the next rebuild drops them (a frame in which something sank ends
        with a rebuild request).  `removed_count` counts them; readbacks skip them."""
        lo, hi = [float(x) for x in min_corner], [float(x) for x in max_corner]
        if len(lo) != 3 or len(hi) != 3 or any(not (a < b) for a, b in zip(lo, hi)):
            raise RejectedInputError(f"sink box needs min < max on three axes, got {lo} / {hi}")
        self._tp.sink_enabled = 1
        for k in range(3):
            self._tp.sink_lo[k], self._tp.sink_hi[k] = lo[k], hi[k]
        self.store.has_sink = True
        self._plan_stale = True

    def clear_sink(self):
        self._tp.sink_enabled = 0
        self._plan_stale = True

    @property
    def removed_count(self) -> int:
        """Particles taken out by the sink so far."""
        return int(self._status.cpu().numpy()[:, 8].sum())

    # -- per frame (pipeline.py:852-880) ------------------------------------------------
    def begin_frame(self):
        self._phase_ms = {k: 0.0 for k in _PHASES}
        self._frame_steps = 0
        self._frame_rebuilds = 0
        self._frame_event_start = len(self.kernel_events)
        self.frame_dts = []       # step sizes of the current frame, in order

    def run_frame(self):
        self._run_frame()
        if self._sunk_pending:
            # lanes emptied by the sink are compacted away by the next rebuild
            self._sunk_pending = False
            self.flags.rebuild_needed = True

    def _run_frame(self):
        self.begin_frame()
        if self.pipelined and self.runtime.n_workers == 1 and \
                self.options.rebuild != "every_step" and not self.options.collect_conservation:
            with torch.cuda.device(self.device):
                if self.cfl_mode and self.device_clock and self.batch_steps > 0:
                    self._run_frame_batched(cfl=True)
                elif self.batch_steps > 0 and not self.cfl_mode:
                    self._run_frame_batched()
                else:
                    self._clock_valid = False
                    self._run_frame_pipelined()
            return
        self._clock_valid = False
        with torch.cuda.device(self.device):
            if self.cfl_mode:
                c_sound = self.material.sound_speed()
                t = 0.0
                while t < self.params.frame_dt - 1e-12:
                    vmax = self.runtime.global_vmax((self._global_step - 2) % 3)
                    self.dt = cfl_dt(vmax + c_sound, self.params, self.params.frame_dt - t)
                    self.run_step(self._global_step)
                    t += self.dt
                    self._frame_steps += 1
                    self.frame_dts.append(self.dt)
            else:
                self.dt = self.params.dt
                for _ in range(self.params.steps_per_frame):
                    self.run_step(self._global_step)
                    self._frame_steps += 1
                    self.frame_dts.append(self.dt)
            if self._pending_gather and not self.lazy_flush:
                self._flush_gather()

    def _run_frame_pipelined(self):
        """run_frame with the host one step ahead of the device.

        Step s+1 is enqueued (guarded) before step s's status block has been read.  When step
        s turns out to have asked for a rebuild, the device skipped step s+1 by itself (guard
        word < s+1), the host restores its bookkeeping and re-issues the step after the
        rebuild -- the same sequence of steps and rebuilds as the reference's
        "read flag, then step" loop (pipeline.py:856-880, 905-940), without a device idle
        gap per step."""
        c_sound = self.material.sound_speed() if self.cfl_mode else 0.0
        frame_dt = self.params.frame_dt
        t = 0.0
        inflight = None          # (slot, step) of the last enqueued, not yet consumed gather
        self._defer = True
        try:
            while True:
                more = (t < frame_dt - 1e-12) if self.cfl_mode else \
                    (self._frame_steps < self.params.steps_per_frame)
                if not more:
                    break
                step = self._global_step
                if self.flags.rebuild_needed:
                    # a rebuild synchronises anyway: drain, then step unguarded
                    if inflight is not None:
                        self._consume(*inflight)
                        inflight = None
                    self._guard = None
                else:
                    self._guard = _capi.Guard(self._guard_word.data_ptr(), step)
                if self.cfl_mode:
                    vmax = self.runtime.global_vmax((step - 2) % 3)
                    self.dt = cfl_dt(vmax + c_sound, self.params, frame_dt - t)
                else:
                    self.dt = self.params.dt
                snap = self._snapshot()
                self._unconsumed = None
                self.step_pre_barrier(step)
                self.runtime.barrier_wait(self.wid)
                self.step_post_barrier(step)
                cur = self._unconsumed
                if inflight is not None:
                    self._consume(*inflight)
                    inflight = None
                    if self.flags.rebuild_needed:
                        # the step just enqueued was skipped on the device: undo it on the host
                        self._restore(snap)
                        self._call("mpm_fill_i32", self._guard_word.data_ptr(), 1, _INT_MAX, _stream_ptr())
                        self.speculative_discards += 1
                        continue
                inflight = cur
                t += self.dt
                self._frame_steps += 1
                self.frame_dts.append(self.dt)
            if inflight is not None:
                self._consume(*inflight)
                if self.flags.rebuild_needed:
                    self._call("mpm_fill_i32", self._guard_word.data_ptr(), 1, _INT_MAX, _stream_ptr())
        finally:
            self._defer = False
            self._guard = None
        if self._pending_gather and not self.lazy_flush:
            self._flush_gather()

    # -- batched steady state (fixed dt): mpm_enqueue_steps ------------------------------------
    def _can_batch(self, next_step=None):
        if self.flags.rebuild_needed:
            return False
        if self._pending_full_clear_parity != -1:
            # the first batch after a rebuild clears the parity the rebuild left untouched itself
            # (mpm_step_plan.full_clear_first); callers that do not say which step comes next
            # (peer.py) take the plain step
            if next_step is None or next_step != self._global_step or \
                    self._pending_full_clear_parity != (next_step & 1):
                return False
        if not self.store.n_groups or self.store.staged_count:
            return False
        if self.options.transfer == "g2p2g":
            return self._fused_active() and self._pending_gather
        return not self._pending_gather

    def _step_plan(self):
        plan = self._plan
        if plan is None or self._plan_stale:
            # buffers may have moved at the last rebuild: the views are refreshed, the rest is static
            st, tb, gr = self.store, self.table, self.grid
            if plan is None:
                plan = _capi.StepPlan()
            plan.store, plan.table = st.view(), tb.view()
            for k in (0, 1):
                plan.raw[k], plan.touched[k] = gr._raw[k].ptr, tb._touched[k].ptr
            plan.vel = gr._vel.ptr
            plan.vel_old = self._vel_old_ptr()
            self._plan_stale = False
        if self._plan is None:
            self._plan = plan
            plan.fused = int(self.options.transfer == "g2p2g")
            plan.status_ring = _RING
            plan.status_dev = self._status.data_ptr()
            plan.status_host = self._status_host.data_ptr()
            for k, ev in enumerate(self._status_events):
                plan.events[k] = ev.cuda_event
            plan.guard_word = self._guard_word.data_ptr()
            plan.fused_margin_lo = FREE_ZONE_LO_CELLS - FUSED_MARGIN_CELLS
            plan.fused_margin_hi = FREE_ZONE_HI_CELLS - 4.0 - FUSED_MARGIN_CELLS
        C.memmove(C.byref(plan.transfer), C.byref(self._params()), C.sizeof(TransferParams))
        gp = self._grid_params()
        gp.fuse_clear = int(self.fuse_clear)
        C.memmove(C.byref(plan.grid), C.byref(gp), C.sizeof(_capi.GridParams))
        return plan

    def _ensure_clock(self):
        """Device step clock of a CFL-auto frame (mpm_step_clock).  Once a device-clocked frame has
        run, the clock already holds the size of the next step (its last grid update computed it)
        and t = 0; it is (re)initialised from the host's vmax ring when steps ran outside it."""
        if self._clock_valid:
            return
        step = self._global_step
        c_sound = self.material.sound_speed()
        dt0 = cfl_dt(self.runtime.global_vmax((step - 2) % 3) + c_sound, self.params, self.params.frame_dt)
        self._clock_host.zero_()
        self._clock_host[step & 1] = dt0
        self._clock.copy_(self._clock_host, non_blocking=True)
        # The update of step `step` reads vmax of step - 1 from the status ring, the one after it
        # vmax of `step`.  The reference's ring has three slots that keep their last value when a
        # step publishes nothing (the first step of a fused run has no gather: slot step % 3 still
        # holds the initial max speed, pipeline.py:866); the same values are planted here.
        s32 = self._status.view(torch.int32)
        for k in (step - 1, step):
            slot = k % _RING
            v2 = np.float32(self.runtime.global_vmax(k % 3)) ** 2
            s32[slot, 1] = int(np.float32(v2).view(np.int32))
            self._slot_clean[slot] = False
        self._clock_valid = True

    def _publish_clock_status(self, step):
        """A device-clocked step without a gather of its own (rebuild step of the fused transfer):
        fetch dt and the frame-end bit the grid update left in the step's status block."""
        slot = step % _RING
        if self._status_alias:
            self._call("mpm_status_publish", self._status_ptr(slot),
                       self._status_alias + slot * _capi.STATUS_BYTES, None, None, _stream_ptr())
        else:
            self._status_host[slot].copy_(self._status[slot], non_blocking=True)
        self._status_events[slot].record()
        self._status_events[slot].synchronize()
        raw = self._status_host.numpy()
        self._last_dt = float(raw.view(np.float64)[slot, 7])
        self._last_frame_end = bool(int(raw.view(np.uint32)[slot, 0]) & _capi.STATUS_FRAME_END)
        self._slot_clean[slot] = False

    def _run_frame_batched(self, cfl=False):
        """Frame with the steady-state steps enqueued in batches from C (mpm_enqueue_steps), two
        batches in flight.  Same guard protocol as _run_frame_pipelined: a step that raises the
        rebuild flag turns every later enqueued step into a no-op on the device; the host drops
        them, rebuilds and carries on from the step after the one that raised the flag -- the
        reference's sequence of steps.

        cfl=True (CFL-auto frames, pipeline.py:856-871): the step sizes live on the device
        (mpm_step_clock).  The host does not know how many steps the frame takes: it keeps
        enqueueing, reads dt and the frame-end bit from each step's status block, and the grid
        update of the step that completes the frame voids the steps enqueued beyond it."""
        spf = self.params.steps_per_frame
        if cfl:
            self._ensure_clock()
            self._use_clock = True
        else:
            self.dt = self.params.dt
        pending = []            # batches in flight: (first_step, n, time-event base or None)
        enq = 0                 # steps of this frame enqueued (confirmed + speculative)
        next_step = self._global_step
        tbase = 0
        frame_done = False
        try:
            while (not frame_done) if cfl else (self._frame_steps < spf):
                while len(pending) < 2 and (cfl or enq < spf) and self._can_batch(next_step):
                    n = self.batch_steps if cfl else min(self.batch_steps, spf - enq)
                    plan = self._step_plan()
                    plan.full_clear_first = int(self._pending_full_clear_parity != -1)
                    self._pending_full_clear_parity = -1
                    tev = None
                    for k in range(2 * n):
                        plan.time_events[k] = None
                    if self.time_kernels:
                        # ONE step of a batch is timed: an event between two kernels of the chain
                        # serialises them fully (no programmatic dependent launch across it), so the
                        # other steps run exactly as they do untimed.  Its position rotates from batch
                        # to batch: the first step after a rebuild (freshly sorted lanes, cold L2) must
                        # not be over-represented in the mean.
                        tk = self._time_rot % n
                        self._time_rot += 1
                        tev = (tbase, tk)
                        plan.time_events[2 * tk] = self._time_events[2 * tbase].cuda_event
                        plan.time_events[2 * tk + 1] = self._time_events[2 * tbase + 1].cuda_event
                        tbase = (tbase + _BATCH) % (2 * _BATCH)
                    # the first step of a batch gathers with the dt of the last grid update done
                    plan.transfer.dt_gather = float(self._vel_dt if not pending else self.dt)
                    self.kernel_calls += 1
                    check(self.lib.mpm_enqueue_steps(C.byref(plan), next_step, n, _stream_ptr()),
                          "mpm_enqueue_steps")
                    pending.append((next_step, n, tev))
                    next_step += n
                    enq += n
                if not pending:
                    # rebuild step, first fused step after a rebuild, pending full clear: one plain step
                    # (its gather's status is read after the whole step is enqueued)
                    self._guard = None
                    self._defer, self._unconsumed = True, None
                    step = self._global_step
                    # a rebuild step may enqueue the batch that follows it from C (mpm_rebuild), so that
                    # the device has work while the host books the new tables
                    left = self.batch_steps if cfl else min(self.batch_steps, spf - self._frame_steps - 1)
                    self._rebuild_next = max(left, 0) if self.flags.rebuild_needed else 0
                    self._rebuild_enqueued = 0
                    try:
                        self.run_step(step)
                    finally:
                        self._defer = False
                        self._rebuild_next = 0
                    if self._unconsumed is not None:
                        self._consume(*self._unconsumed)
                        self._unconsumed = None
                    elif cfl:
                        self._publish_clock_status(step)
                    if cfl:
                        self.dt = self._vel_dt = self._last_dt
                        frame_done = self._last_frame_end
                    self._frame_steps += 1
                    self.frame_dts.append(self.dt)
                    enq = self._frame_steps
                    next_step = self._global_step
                    if self._rebuild_enqueued:
                        n = self._rebuild_enqueued
                        self._rebuild_enqueued = 0
                        self._pending_full_clear_parity = -1      # that batch cleared the other parity
                        if self.flags.rebuild_needed or frame_done:
                            # the rebuild step itself asked for another rebuild / ended the frame: its
                            # gather raised the guard, the batch behind it ran as no-ops
                            self.speculative_discards += n
                            self._pending_full_clear_parity = (step + 1) & 1
                            if self.flags.rebuild_needed and self._rebuild_tail_ok_static():
                                self._guard_reset_in_rebuild = True
                            else:
                                self._call("mpm_fill_i32", self._guard_word.data_ptr(), 1, _INT_MAX, _stream_ptr())
                        else:
                            pending.append((next_step, n, None))
                            next_step += n
                            enq += n
                    continue
                first, n, tev = pending.pop(0)
                for k in range(n):
                    step = first + k
                    self._slot_clean[step % _RING] = False
                    self._consume(step % _RING, step)
                    if cfl:
                        self.dt = self._last_dt
                        frame_done = self._last_frame_end
                    if tev is not None and k == tev[1]:
                        name = "mpm_g2p2g" if self.options.transfer == "g2p2g" else "mpm_p2g"
                        # read now: the ring's events are recorded again by the batch after next (the
                        # step's status arrived, so its transfer kernel and both events are complete)
                        ms = self._time_events[2 * tev[0]].elapsed_time(self._time_events[2 * tev[0] + 1])
                        self.kernel_events.append((name, _Ms(ms, self.flags.steps_since_rebuild), None))
                    # step `step` itself ran to completion (the guard only stops LATER steps)
                    self._global_step = step + 1
                    self._vel_dt = self.dt
                    self.flags.steps_since_rebuild += 1
                    self.runtime.generations += 1
                    self._frame_steps += 1
                    self.frame_dts.append(self.dt)
                    if self.flags.rebuild_needed or frame_done:
                        self.speculative_discards += (n - 1 - k) + sum(b[1] for b in pending)
                        pending = []
                        enq = self._frame_steps
                        next_step = self._global_step
                        if self.flags.rebuild_needed and self._rebuild_tail_ok_static():
                            # nothing guarded is enqueued before the rebuild this flag asks for, and
                            # mpm_rebuild resets the word itself (one launch and its gap less)
                            self._guard_reset_in_rebuild = True
                        else:
                            self._call("mpm_fill_i32", self._guard_word.data_ptr(), 1, _INT_MAX, _stream_ptr())
                        break
        finally:
            self._use_clock = False
        if self._pending_gather and not self.lazy_flush:
            self._flush_gather()

    def _snapshot(self):
        f = self.flags
        return (self._pending_gather, self._pending_full_clear_parity, self._vel_dt,
                f.steps_since_rebuild, f.fused_mode, self._global_step, self._fused_now,
                self.runtime.generations, list(self._slot_clean), len(self.kernel_events))

    def _restore(self, snap):
        f = self.flags
        (self._pending_gather, self._pending_full_clear_parity, self._vel_dt,
         f.steps_since_rebuild, f.fused_mode, self._global_step, self._fused_now,
         self.runtime.generations, clean, n_events) = snap
        self._slot_clean = clean
        del self.kernel_events[n_events:]

    # -- one step, split around the barrier (pipeline.py:905-940) --------------------------
    def step_pre_barrier(self, step):
        par = step & 1
        if self.options.rebuild == "every_step":
            self.flags.rebuild_needed = True
        rebuilt = False
        if self.flags.rebuild_needed:
            flushed = None
            if self._pending_gather:
                # the flush's status block is read at the rebuild's first host sync, not before
                # its first kernels are enqueued (one device idle gap less per rebuild)
                flushed = self._flush_gather(defer=True)
            self._rebuild(step, par, flushed, tail=self._rebuild_tail_ok())
            rebuilt = True
        else:
            self._clear(par)
        fused_now = self._fused_active()
        self.flags.fused_mode = fused_now
        if self._tail_done:
            pass        # mpm_rebuild issued the P2G (and the grid update) of this step itself
        elif fused_now and self._pending_gather:
            self._run_g2p2g(step, par)
        else:
            if self._pending_gather:
                self._flush_gather()
            self._run_p2g(step, par)
        self._publish(par, rebuilt)
        self._fused_now = fused_now

    def step_post_barrier(self, step):
        par = step & 1
        self._post_barrier(par)
        self._reduce_and_update(par, step)
        if self._fused_now:
            self._pending_gather = True
        elif self._tail_g2p_done:
            # issued (and its status block published) by mpm_rebuild behind the grid update
            self._tail_g2p_done = False
            slot = step % _RING
            self._slot_clean[slot] = False
            if self._defer:
                self._unconsumed = (slot, step)
            else:
                self._consume(slot, step)
            self._pending_gather = False
        else:
            self._run_g2p(step)
            self._pending_gather = False
        self.flags.steps_since_rebuild += 1
        self._global_step = step + 1

    def run_step(self, step):
        if not self._use_clock:
            self._clock_valid = False      # a step with a host-given dt: the device clock is stale
        with torch.cuda.device(self.device):
            self.step_pre_barrier(step)
            self.runtime.barrier_wait(self.wid)
            self.step_post_barrier(step)

    # -- phases ---------------------------------------------------------------------------
    def _fused_active(self):
        if self.options.transfer != "g2p2g":
            return False
        if self.store.staged_count:
            return False
        if self.store.count >= self.options.fused_threshold:
            # pipeline.py:948-954: the fallback is announced once per worker
            if not self._fused_fallback_logged:
                log.info("worker %d: %d particles exceed the fused-transfer threshold of %d; "
                         "using split transfers", self.wid, self.store.count,
                         self.options.fused_threshold)
                self._fused_fallback_logged = True
            return False
        return True

    @property
    def effective_transfer(self) -> str:
        """The transfer arm the worker is actually running ("g2p2g" falls back to "split" above
        PipelineOptions.fused_threshold particles and while appends are staged)."""
        if self.options.transfer != "g2p2g" or self.store.count >= self.options.fused_threshold:
            return "split"
        return "g2p2g"

    def _rebuild_tail_ok_static(self):
        cls = type(self)
        return (self.runtime.n_workers == 1
                and cls._publish is CudaWorker._publish
                and cls._reduce_and_update is CudaWorker._reduce_and_update
                and cls._run_p2g is CudaWorker._run_p2g
                and not self.options.collect_conservation and not self.params.flip_blend > 0.0)

    def _rebuild_tail_ok(self):
        """A single worker lets mpm_rebuild issue the rest of the rebuild step (P2G, grid update)
        behind the rebuild kernels; workers with peers publish / meet / re-tag in between."""
        return self._guard is None and self._rebuild_tail_ok_static()

    def _rebuild(self, step, par, flushed=None, tail=False):
        """Worker._rebuild (pipeline.py:958-1015) on the device: one call (mpm_rebuild) that enqueues
        every rebuild kernel WITHOUT a host round trip in between (the counts stay on the device,
        launches are sized by the capacities given here), then -- for a single worker (`tail`) --
        the rest of the rebuild step and the first batch of steady steps.  The host waits only
        for the scalars (mpm_rebuild_wait), while those kernels run, and does its bookkeeping
        of the new tables under their cover.  Buffers stay Python's: they are sized here from
        the counts of the previous rebuild (4x growth rule, so a steady state never
        reallocates); a count that outgrew one aborts the chain on the device and the call
        reports what it needs."""
        lib, st, tb, gr = self.lib, self.store, self.table, self.grid
        stream = _stream_ptr()
        t_rebuild = time.perf_counter()
        staged, staged_ids, n_staged = st.take_staged()
        n_upper = st.count + n_staged
        S, S64 = self._scratch_i32, self._scratch_i64
        nxt = 1 - st.cur
        new_bufs = [b[nxt] for b in (st._data, st._orig_id, st._lane_meta, st._group_len, st._group_block,
                                     st._group_start, st._group_ctx)]
        # requests: the counts of the last rebuild (a first guess for the very first one)
        want_g = max(tb.n_gblocks, 1)
        want_groups = max(st.n_groups, n_upper // 32 + 1)
        want_nodes = max(tb.count, 1)
        # hash capacity: load factor < 1/8 against the pblock count seen last time, or a
        # conservative first guess; an overflow quadruples it and retries
        cap = max(tb.hash_cap, _pow2_at_least(8 * max(tb.count, 1)), 1 << 12)
        if tb.count == 0:
            cap = max(cap, _pow2_at_least(max(n_upper // 2, 1)))
        tight = True
        # The plan of the last rebuild out of this half of the store is reused as it stands when
        # nothing it describes can have changed: no staged particles, the same particle count, no
        # buffer reallocated since (only the step-dependent fields below are refreshed).  Its launch
        # bounds may then be older than the counts; a count that outgrew one aborts on the device and
        # comes back through the sizing below, like any other.
        # graph replay only for a scene in steady state (same particle count, no buffer moved over the
        # last rebuilds): a scene whose count changes all the time (emitter, sink) would capture a
        # graph per shape and never reuse it.  `by_capacity`: the old store described by the capacity
        # of its buffers and its count on the device (what makes the chain replayable) -- only then,
        # since it also launches the compaction over the whole capacity.
        shape = (n_upper, n_staged, DeviceBuffer.generation)
        self._rb_stable = self._rb_stable + 1 if shape == self._rb_shape else 0
        self._rb_shape = shape
        by_capacity = bool(self.rebuild_graph and n_staged == 0 and n_upper <= self.rebuild_graph_max
                           and self._rb_stable >= 3 and st.n_groups > 0 and self._ngroups_dev_valid[st.cur])
        use_graph = by_capacity and self._rb_stable >= 4
        ck = (st.cur, n_upper, DeviceBuffer.generation, tb.hash_cap, by_capacity) \
            if (n_staged == 0 and st.n_groups > 0) else None
        cached = self._rb_cache.get(st.cur) if ck is not None else None
        fast = cached is not None and cached[0] == ck
        if fast and not by_capacity:
            # the reused plan states the old store's group count by value: refresh it (and make sure
            # the compaction scratch, sized for the count of the rebuild the plan was made for, holds it)
            if self._scratch["glive"].capacity < st.n_groups + 1:
                fast = False
            else:
                cached[1].old_store.n_groups = st.n_groups
        if fast:
            plan, res = cached[1], cached[2]
        else:
            plan, res = _capi.RebuildPlan(), _capi.RebuildResult()
            self._rebuild_static_fields(plan, st, nxt, n_upper, n_staged, staged, staged_ids, by_capacity)
        cur_before = st.cur
        plan.use_graph = int(use_graph)
        self._rebuild_step_fields(plan, step, par, tail)
        next_n = self._rebuild_next_n
        while True:
            if fast:
                plan.raw_par = gr._raw[par].ptr
                plan.touched_par = tb._touched[par].ptr
            else:
                self._rebuild_size(plan, par, want_g, want_groups, want_nodes, cap, tight, new_bufs, n_upper)
            if next_n > 0:
                self._plan_stale = True              # buffers may just have been grown
                sp = self._step_plan()
                sp.full_clear_first = 1              # step + 1 is the first use of the other parity
                sp.transfer.dt_gather = float(self.dt)
                for k in range(2 * next_n):
                    sp.time_events[k] = None
                plan.next_steps = C.addressof(sp)
                plan.next_first_step, plan.next_n_steps = int(step) + 1, next_n
            else:
                plan.next_steps = None
                plan.next_first_step = plan.next_n_steps = 0
            self.kernel_calls += 1
            rc = lib.mpm_rebuild(C.byref(plan), C.byref(res), stream)
            if flushed is not None:
                self._consume(*flushed)      # the gather flushed just before this rebuild
                flushed = None
            if rc == 0 and plan.async_:
                rc = lib.mpm_rebuild_wait(C.byref(plan), C.byref(res))
            if rc == _capi.NEED_CAPACITY:
                if res.need_hash:
                    cap *= 4
                want_g = max(want_g, res.need_gblocks, (res.need_table + 26) // 27)
                want_groups = max(want_groups, res.need_groups)
                want_nodes = max(want_nodes, res.need_nodes)
                tight = False
                fast = False
                continue
            if rc == -2 and res.bad_particle != _INT_MAX:
                raise SpatialDomainError(
                    f"worker {self.wid}: particle {res.bad_particle} of the rebuild input lies outside "
                    f"the encodable domain [0, 2^21) cells")
            if rc == -2 and res.bad_block != _INT_MAX:
                code = int(self._scratch["gcodes"].data[res.bad_block].item())
                x, y, z = _decode(code)
                raise SpatialDomainError(
                    f"block ({x - CELL_BIAS // 4}, {y - CELL_BIAS // 4}, {z - CELL_BIAS // 4}) "
                    f"touches the domain boundary; scenes must leave a one-block margin")
            check(rc, "mpm_rebuild")
            break
        self._rebuild_adopt(res, nxt, new_bufs, step, par, t_rebuild)
        if n_staged == 0:
            self._rb_cache[cur_before] = ((cur_before, n_upper, DeviceBuffer.generation, tb.hash_cap, by_capacity),
                                          plan, res)

    def _rebuild_static_fields(self, plan, st, nxt, n_upper, n_staged, staged, staged_ids, by_capacity):
        """Fields of a rebuild plan that only change with the buffers, the particle count or staging."""
        S, S64 = self._scratch_i32, self._scratch_i64
        plan.old_store = st.view()
        old_bufs = [b[st.cur] for b in (st._data, st._orig_id, st._lane_meta, st._group_len, st._group_block,
                                        st._group_start, st._group_ctx)]
        old_bound = st.n_groups
        if by_capacity:
            # the old store by its CAPACITY, its count read on the device: the chain then looks the
            # same from one rebuild to the next (mpm_rebuild replays it as a graph)
            old_bound = min(b.capacity for b in old_bufs)
            plan.old_store.n_groups = old_bound
            plan.old_store.n_groups_dev = self._ngroups_dev.data_ptr() + 4 * st.cur
        plan.n_groups_out = self._ngroups_dev.data_ptr() + 4 * nxt
        plan.use_graph = 0        # set per call (_rebuild): only once the shape has been stable for a while
        plan.n_staged, plan.n_upper = n_staged, n_upper
        plan.staged = staged.data_ptr() if n_staged else None
        plan.staged_ids = staged_ids.data_ptr() if n_staged else None
        plan.dx = float(self.params.dx)
        plan.glive = S("glive", old_bound + 1).ptr
        for tag in ("src_slot", "pslot", "flag", "gidx", "tmp_perm", "perm"):
            setattr(plan, tag, S(tag, n_upper).ptr)
        plan.codes, plan.gcodes = S64("codes", n_upper).ptr, S64("gcodes", n_upper).ptr
        scan = S("scan", n_upper // 8 + 1024)                # block sums of the largest scan
        plan.scan = scan.ptr
        plan.node_bytes = self._node_bytes
        plan.scalars_dev, plan.scalars_host = self._scalars.data_ptr(), self._scalars_host.data_ptr()
        plan.large_list = S("large_list", n_upper // 1024 + 2).ptr

    def _rebuild_step_fields(self, plan, step, par, tail):
        """Fields of a rebuild plan that depend on the step: the guard, the rest of the rebuild step and
        the batch behind it (every one of them is assigned, a reused plan keeps nothing)."""
        plan.guard_word, plan.guard_step = None, 0
        plan.p2g_params = plan.grid_params = plan.p2g_status = plan.grid_reset_status = None
        plan.g2p_params = plan.g2p_status = plan.status_publish_dst = plan.status_event = None
        plan.async_, plan.done_event = 0, None
        if self._guard_reset_in_rebuild or tail:
            # tail: nothing guarded is in flight (_rebuild_tail_ok), the word is reset by the call and
            # then guards the rest of the step and the next batch, so that an aborted rebuild (a
            # buffer too small) voids them without the host
            plan.guard_word = self._guard_word.data_ptr()
            plan.guard_step = int(step)
            self._guard_reset_in_rebuild = False
        next_n = 0
        if tail:
            # rest of the step (step_pre_barrier / step_post_barrier): P2G into status slot `step`,
            # grid update that also zeroes the status block of the gather following it
            fused = self._fused_active()
            # private copies: _step_plan() below refills the cached structs for the next batch
            tp, gp = self._tp_scatter, self._gp_tail
            C.memmove(C.byref(tp), C.byref(self._params(step=step)), C.sizeof(TransferParams))
            C.memmove(C.byref(gp), C.byref(self._grid_params(step)), C.sizeof(_capi.GridParams))
            gp.fuse_clear = int(self.fuse_clear)
            reset_slot = (step + 1 if fused else step) % _RING
            plan.p2g_params, plan.grid_params = C.addressof(tp), C.addressof(gp)
            plan.p2g_status = self._status_ptr(step % _RING)
            plan.grid_reset_status = self._status_ptr(reset_slot)
            self._tail_reset_slot = reset_slot
            plan.async_ = 1
            plan.done_event = self._rebuild_event.cuda_event
            if not fused and self._status_alias and not self.profile_all_phases:
                # split transfer: the step's gather and the publication of its status block too
                slot = step % _RING
                g2 = self._tp_gather
                C.memmove(C.byref(g2), C.byref(tp), C.sizeof(TransferParams))
                g2.dt_gather = float(self.dt)          # the update of this very step (pipeline.py:1230)
                g2.clock_gather_step = int(step)
                plan.g2p_params = C.addressof(g2)
                plan.g2p_status = self._status_ptr(slot)
                plan.status_publish_dst = (self._status_alias + slot * _capi.STATUS_BYTES) \
                    if self._status_alias else None
                plan.status_event = self._status_events[slot].cuda_event
            next_n = int(self._rebuild_next or 0)
            if next_n > 0 and (plan.g2p_params or fused):
                # the first batch of steady steps, enqueued by the call itself behind the rebuild step
                # (its store / table views are filled in C from this rebuild)
                self._plan_stale = True
            else:
                next_n = 0
        self._rebuild_next_n = next_n

    def _rebuild_size(self, plan, par, want_g, want_groups, want_nodes, cap, tight, new_bufs, n_upper):
        """Size the caller-owned buffers of a rebuild (4x growth rule) and describe them to the plan."""
        st, tb, gr = self.store, self.table, self.grid
        S = self._scratch_i32
        scan = self._scratch["scan"]
        # block-indexed scratch and tables; codes/origin/touched sized for the worst case of the
        # dilation, 27 n_g (they are small)
        qslot, qflag = S("qslot", 27 * want_g), S("qflag", 2 * 27 * want_g)
        bin_start, bgf = S("bin_start", want_g * 64 + 1), S("bgf", want_g + 1)
        tb.ensure_hash(cap)
        tb._codes.ensure_capacity(27 * want_g, keep=False)
        tb._origin.ensure_capacity(27 * want_g, keep=False)
        tb._neighbor.ensure_capacity(want_g, keep=False)
        for k in (0, 1):
            tb._touched[k].len = min(tb._touched[k].len, tb.count)
            tb._touched[k].ensure_capacity(27 * want_g, keep=True)
        for buf in new_bufs:
            buf.ensure_capacity(want_groups, keep=False)
        gr._vel.ensure_capacity(want_nodes, keep=False)
        gr._raw[par].ensure_capacity(want_nodes, keep=False)
        gr._raw[1 - par].ensure_capacity(want_nodes, keep=False)   # next step's parity: cleared in full there
        plan.qslot, plan.qflag, plan.bin_start, plan.bgf = qslot.ptr, qflag.ptr, bin_start.ptr, bgf.ptr
        # Capacities double as launch bounds (the counts are read on the device).  The 4x growth
        # rule leaves them up to 4x the real counts; twice the last counts is what a first attempt
        # launches over, the full capacity only after a count outgrew that.
        plan.cap_gblocks = min(tb._neighbor.capacity, qslot.capacity // 27, qflag.capacity // 54,
                               (bin_start.capacity - 1) // 64, bgf.capacity - 1,
                               (scan.capacity - 2) * 16,     # 64 bins per block, 1024 per scan tile
                               _pow2_at_least(max(2 * want_g, 64)) if tight else _INT_MAX)
        plan.hkeys, plan.hvals, plan.hfirst = tb._hkeys.ptr, tb._hvals.ptr, tb._hfirst.ptr
        plan.hash_cap = cap
        plan.cap_table = min(tb._codes.capacity, tb._origin.capacity, tb._touched[0].capacity,
                             tb._touched[1].capacity)
        plan.table_codes, plan.table_origin = tb._codes.ptr, tb._origin.ptr
        plan.table_neighbor = tb._neighbor.ptr
        plan.new_store = StoreView(*(b.ptr for b in new_bufs[:6]), 0, st.nch, new_bufs[6].ptr)
        plan.cap_groups = min(b.capacity for b in new_bufs)
        plan.vel, plan.raw_par = gr._vel.ptr, gr._raw[par].ptr
        plan.touched_par = tb._touched[par].ptr
        plan.cap_nodes = min(gr._vel.capacity, gr._raw[par].capacity, gr._raw[1 - par].capacity,
                             _pow2_at_least(max(2 * want_nodes, 256)) if tight else _INT_MAX)

    def _rebuild_adopt(self, res, nxt, new_bufs, step, par, t_rebuild):
        """Host bookkeeping of the tables a rebuild produced."""
        st, tb, gr = self.store, self.table, self.grid
        n, n_g, count, G = res.n, res.n_gblocks, res.count, res.n_groups
        self._ngroups_dev_valid[nxt] = True
        self.rebuild_graph_replays += int(res.graph == 2)
        tb.n_gblocks, tb.count = n_g, count
        tb._codes.len = tb._origin.len = count
        tb._neighbor.len = n_g
        for buf in new_bufs:
            buf.len = G
        st.cur, st.n_groups, st.count = nxt, G, n
        self.last_perm = self._scratch["perm"].data[:n]
        self.last_gidx = self._scratch["gidx"].data[:n]
        # nodal buffers (pipeline.py:996-1006): vel and raw[par] were zeroed by the call; the other
        # parity keeps whatever it held and is cleared in full at its next use
        gr._vel.len = gr._raw[par].len = count
        gr._raw[1 - par].resize(count, keep=False)
        if gr._vel_old is not None:
            gr._vel_old.resize(count, keep=False)
        gr.count = count
        for k in (0, 1):
            tb._touched[k].len = count
        self._tail_done = bool(res.tail_done)
        self._tail_g2p_done = bool(res.g2p_done)
        self._rebuild_enqueued = int(res.next_done)
        self._pending_full_clear_parity = 1 - par
        self._plan_stale = True       # buffers may have moved: the batched-step plan refreshes its views
        self._published_codes = (tb._codes, count)
        self.flags.rebuild_needed = False
        self.flags.steps_since_rebuild = 0
        self.rebuild_steps.append(step)
        self._frame_rebuilds += 1
        self._phase_ms["rebuild"] += (time.perf_counter() - t_rebuild) * 1e3

    def _clear(self, par):
        """Worker._clear (pipeline.py:1022-1037)."""
        count = self.table.count
        if not count:
            return
        full = int(self._pending_full_clear_parity == par)
        if full:
            self._pending_full_clear_parity = -1
        elif self.fuse_clear and self.runtime.n_workers == 1:
            return   # rows were zeroed by the grid update that consumed them
        self._call("mpm_clear", self.grid._raw[par].ptr, self.table._touched[par].ptr, count, full,
                   self._node_bytes, self._gref(), _stream_ptr())

    def _params(self, margin_shrink=0.0, step=0, gather_step=0):
        tp = self._tp
        tp.dt = float(self.dt)
        tp.dt_gather = float(self._vel_dt)
        tp.margin_lo = FREE_ZONE_LO_CELLS - margin_shrink
        tp.margin_hi = FREE_ZONE_HI_CELLS - 4.0 - margin_shrink
        # device-clocked CFL frame: dt / dt_gather above are ignored, the kernels read the clock
        tp.clock = self._clock.data_ptr() if self._use_clock else None
        tp.clock_step, tp.clock_gather_step = int(step), int(gather_step)
        return tp

    def _vel_old_ptr(self):
        if self.params.flip_blend > 0.0:
            gr = self.grid
            if gr._vel_old is None:
                gr._vel_old = DeviceBuffer(torch.float32, (64, 4), self.device)
            gr._vel_old.resize(self.table.count, keep=True)
            return gr._vel_old.ptr
        return None

    def _gref(self):
        return C.byref(self._guard) if self._guard is not None else None

    def _status_ptr(self, slot):
        return self._status.data_ptr() + slot * _capi.STATUS_BYTES

    def _run_p2g(self, step, par):
        st = self.store
        if not st.n_groups:
            return
        sv, tv = st.view(), self.table.view()
        self._call("mpm_p2g", C.byref(sv), C.byref(tv), self.grid._raw[par].ptr,
                   self.table._touched[par].ptr, C.byref(self._params(step=step)),
                   self._status_ptr(step % _RING), self._gref(), _stream_ptr())

    def _gather_slot(self, step, stream):
        slot = step % _RING
        if not self._slot_clean[slot]:
            self._call("mpm_status_reset", self._status_ptr(slot), self._gref(), stream)
        self._slot_clean[slot] = False
        return slot

    def _after_gather(self, slot, step):
        if self._status_alias:
            self._call("mpm_status_publish", self._status_ptr(slot),
                       self._status_alias + slot * _capi.STATUS_BYTES, None, None, _stream_ptr())
        else:
            self._status_host[slot].copy_(self._status[slot], non_blocking=True)
        self._status_events[slot].record()
        if self._defer:
            self._unconsumed = (slot, step)
        else:
            self._consume(slot, step)

    def _run_g2p(self, step):
        st = self.store
        if not st.n_groups:
            self.runtime.publish_vmax(step % 3, self.wid, 0.0)
            return
        sv, tv = st.view(), self.table.view()
        stream = _stream_ptr()
        slot = self._gather_slot(step, stream)
        self._call("mpm_g2p", C.byref(sv), C.byref(tv), self.grid._vel.ptr, self._vel_old_ptr(),
                   C.byref(self._params(step=step, gather_step=step)), self._status_ptr(slot),
                   self._gref(), stream)
        self._after_gather(slot, step)

    def _ensure_flushed(self):
        """Called by the particle store before anything reads or writes particle state."""
        if self._pending_gather and self.lazy_flush and not self._flushing:
            self._flushing = True
            try:
                with torch.cuda.device(self.device):
                    self._flush_gather()
            finally:
                self._flushing = False

    def _flush_gather(self, defer=False):
        """Complete a pending fused gather.  Its status block is read back at once, or (defer)
        handed to the caller as (slot, step) to be consumed at its next host sync."""
        guard, was_defer, unconsumed = self._guard, self._defer, self._unconsumed
        use_clock = self._use_clock
        self._guard, self._defer = None, bool(defer)
        self._unconsumed = None
        self._use_clock = False      # the flushed step's dt has been read back: _vel_dt, by value
        try:
            self._run_g2p(self._global_step)
            flushed = self._unconsumed
        finally:
            self._guard, self._defer, self._unconsumed = guard, was_defer, unconsumed
            self._use_clock = use_clock
        self._pending_gather = False
        return flushed

    def _run_g2p2g(self, step, par):
        st = self.store
        if not st.n_groups:
            return
        sv, tv = st.view(), self.table.view()
        stream = _stream_ptr()
        slot = self._gather_slot(step, stream)
        self._call("mpm_g2p2g", C.byref(sv), C.byref(tv), self.grid._vel.ptr, self._vel_old_ptr(),
                   self.grid._raw[par].ptr, self.table._touched[par].ptr,
                   C.byref(self._params(FUSED_MARGIN_CELLS, step=step, gather_step=step - 1)),
                   self._status_ptr(slot), self._gref(), stream)
        self._after_gather(slot, step)

    def _consume(self, slot, step):
        """Read the status block written by a gather: free-zone flag -> rebuild_needed,
        max speed -> vmax ring (pipeline.py:1102-1104), addressing counter -> exception
        (pipeline.py:1233-1238)."""
        self._status_events[slot].synchronize()
        views = self._status_views
        if views is None:
            # numpy views of the pinned ring, made once: this runs for every substep
            raw = self._status_host.numpy()
            views = self._status_views = (raw, raw.view(np.uint32), raw.view(np.float32))
        raw, u32, f32 = views
        word = int(u32[slot, 0])
        if word & _capi.STATUS_ZONE:
            self.flags.rebuild_needed = True
        if self._tp.sink_enabled:
            removed = int(raw[slot, 8])          # accumulates per slot
            if removed != self._removed_seen[slot]:
                self._removed_seen[slot] = removed
                self._sunk_pending = True
        if self._use_clock:
            self._last_dt = float(raw.view(np.float64)[slot, 7])
            self._last_frame_end = bool(word & _capi.STATUS_FRAME_END)
        vmax2 = float(f32[slot, 1])
        self.runtime.publish_vmax(step % 3, self.wid, math.sqrt(max(vmax2, 0.0)))
        if raw[slot, 1 + C_ADDRESS_ERR]:
            raise ContractViolationError(
                f"worker {self.wid}: {int(raw[slot, 1 + C_ADDRESS_ERR])} stencil accesses left the "
                f"27-neighbor pblock set")

    def _check_addressing(self):
        c = self.counters
        if c[C_ADDRESS_ERR]:
            raise ContractViolationError(
                f"worker {self.wid}: {int(c[C_ADDRESS_ERR])} stencil accesses left the "
                f"27-neighbor pblock set")

    def _publish(self, par, rebuilt):
        codes, count = self._published_codes
        self.runtime.publish_step(par, self.wid, dict(
            raw=self.grid._raw[par], touched=self.table._touched[par], codes=codes,
            code_count=count, rebuilt=rebuilt))

    def _post_barrier(self, par):
        """Shared-block tagging on rebuild steps (pipeline.py:1147-1164)."""
        n = self.runtime.n_workers
        if n == 1:
            return
        states = [self.runtime.peer_step(par, q) for q in range(n)]
        if any(s["rebuilt"] for s in states):
            stream = _stream_ptr()
            for q, s in enumerate(states):
                if q == self.wid:
                    continue
                m = self._peer_map[q]
                if m is None:
                    m = self._peer_map[q] = DeviceBuffer(torch.int32, (), self.device)
                m.resize(self.table.count, keep=False)
                self._call("mpm_tag_shared", s["codes"].ptr, int(s["code_count"]),
                           self.table._hkeys.ptr, self.table._hvals.ptr, self.table.hash_cap,
                           m.ptr, self.table.count, stream)
        self._peer_states = states

    def _reduce_and_update(self, par, step=None):
        """pipeline.py:1166-1231 in one kernel: reduce over peers, finalize, boundary."""
        if step is None:
            step = self._global_step
        if self._tail_done:
            # issued by mpm_rebuild behind the P2G of this (rebuild) step
            self._tail_done = False
            self._slot_clean[self._tail_reset_slot] = True     # the slot that update zeroed
            self._vel_dt = self.dt
            return
        tb, gr = self.table, self.grid
        count = tb.count
        stream = _stream_ptr()
        peers = []
        if self.runtime.n_workers > 1 and self._peer_states is not None:
            for q, s in enumerate(self._peer_states):
                if q == self.wid or self._peer_map[q] is None:
                    continue
                peers.append((s["raw"].ptr, s["touched"].ptr, self._peer_map[q].ptr))
        if self.options.collect_conservation:
            self._collect_conservation(par)
        gp = self._grid_params(step)
        gp.fuse_clear = int(self.fuse_clear and self.runtime.n_workers == 1)
        gp.n_peers = len(peers)
        for k, (r, t, m) in enumerate(peers):
            gp.peer_raw[k], gp.peer_touched[k], gp.peer_map[k] = r, t, m
        tv = tb.view()
        if count:
            # the update also zeroes the status block of the gather that follows it in stream
            # order: this step's G2P, or the next step's fused gather / the frame-end flush
            nxt = (step + 1 if self._fused_now else step) % _RING
            self._grid_update_launch(gp, tv, par, self._status_ptr(nxt), stream)
            self._slot_clean[nxt] = True
        self._vel_dt = self.dt

    def _grid_params(self, step=None):
        """mpm_grid_params with the per-run constants filled once; dt set per call."""
        gp = self._gp
        if gp is None:
            gp = self._gp = _capi.GridParams()
            for k in range(3):
                gp.gravity[k] = float(self.params.gravity[k])
            bc = self.boundary
            gp.apply_bc = int(bc is not None)
            if bc is not None:
                gp.bc_sticky = int(bc.mode == "sticky")
                for k in range(3):
                    gp.box_lo[k] = float(bc.min_corner[k])
                    gp.box_hi[k] = float(bc.max_corner[k])
            gp.dx = float(self.params.dx)
        gp.dt = float(self.dt)
        gp.deterministic = int(bool(self.options.deterministic))
        gp.block_filter = 0
        gp.fuse_clear = 0
        gp.n_peers = 0
        if self._use_clock:
            # device-clocked CFL frame (mpm_step_clock): the update advances the clock
            gp.clock = self._clock.data_ptr()
            gp.vmax_ring, gp.vmax_ring_len = self._status.data_ptr(), _RING
            gp.frame_dt = float(self.params.frame_dt)
            gp.cfl_dx = float(self.params.cfl * self.params.dx)
            gp.c_sound = float(self.material.sound_speed())
            gp.n_vmax_peers = 0
            if step is not None:      # batches: mpm_enqueue_steps sets these per step
                gp.clock_step = int(step)
                gp.clock_status = self._status_ptr(int(step) % _RING)
        else:
            gp.clock = None
        return gp

    def _grid_update_launch(self, gp, tv, par, reset_ptr, stream):
        tb, gr = self.table, self.grid
        self._call("mpm_grid_update", gr._raw[par].ptr, tb._touched[par].ptr, gr._vel.ptr,
                   self._vel_old_ptr(), C.byref(tv), C.byref(gp), reset_ptr, self._gref(), stream)

    def _collect_conservation(self, par):
        """(pm, pmom x3, gm, gmom x3) rows of pipeline.py:1189-1203 (own raw rows only)."""
        out = torch.zeros(4, dtype=torch.float64, device=self.device)
        self._call("mpm_grid_aggregates", self.grid._raw[par].ptr, self.table._touched[par].ptr,
                   self.table.count, int(self.options.deterministic), out.data_ptr(), _stream_ptr())
        p = self.store._aggregates()
        g = out.cpu().numpy()
        self.conservation.append((p[0], p[1], p[2], p[3], g[0], g[1], g[2], g[3]))


def _decode(code: int):
    def compact(v):
        v &= 0x1249249249249249
        v = (v ^ (v >> 2)) & 0x10C30C30C30C30C3
        v = (v ^ (v >> 4)) & 0x100F00F00F00F00F
        v = (v ^ (v >> 8)) & 0x1F0000FF0000FF
        v = (v ^ (v >> 16)) & 0x1F00000000FFFF
        v = (v ^ (v >> 32)) & 0x1FFFFF
        return v
    return compact(code), compact(code >> 1), compact(code >> 2)


def make_single_worker(particles, velocities, material, params, boundary, mass, device=None,
                       **options):
    """The reference tests' harness (tests/conftest.py:18-38 of the reference) for the CUDA
    worker: a solo runtime + worker, seeded and ready for `w.run_step(s)`."""
    from .multiworker import SharedRuntime
    particles = np.asarray(particles)
    velocities = np.asarray(velocities)
    worker_kw = {k: options.pop(k) for k in ("count_stats", "fuse_clear") if k in options}
    vmax = float(np.linalg.norm(velocities, axis=1).max()) if len(velocities) else 0.0
    runtime = SharedRuntime(1, initial_vmax=vmax)
    w = CudaWorker(0, runtime, params, material, boundary, PipelineOptions(**options),
                   device=device, **worker_kw)
    w.seed_particles(particles, velocities, mass, ids=np.arange(len(particles), dtype=np.int64))
    w.dt = params.dt
    return w
