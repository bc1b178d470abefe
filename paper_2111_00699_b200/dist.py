"""One process per GPU: spatial partition of the particles, halo rows exchanged over NCCL.

The reference scales by giving each worker a contiguous slab of particles (stable argsort
along the longest axis, multiworker.py:114-137); every worker owns its block table and nodal
buffers, and the only cross-worker data are the raw nodal rows of blocks that two workers
both hold (pipeline.py:1172-1188), read once per step after the single barrier.  With one
process per GPU the same protocol becomes:

  per step   all_gather of 4 ints per rank (rebuilt flag, block count, max speed bits, step)
             -- this is the step's barrier and feeds the CFL vmax ring with the reference's
             two-step lag (pipeline.py:859-867);
  on rebuild all_gather of the block-code lists, shared-block tagging on the device
             (mpm_tag_shared) and send/recv row lists, both ordered by the receiver's block
             index so that no index list crosses the wire;
  per step   mpm_pack_halo per peer -> batched isend/irecv of the packed rows on a
             communication stream, while mpm_grid_update(block_filter=1) updates the blocks no
             peer holds on the compute stream; then mpm_grid_update(block_filter=2) adds the
             received rows and updates the halo blocks.

The transport is torch.distributed (NCCL on GPUs).  With the gloo backend (CPU tests, or two
ranks sharing one GPU in the single-GPU check) tensors are staged through host memory.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from .multiworker import partition_particles
from .worker import _RING, CudaWorker, _stream_ptr
from .memory import DeviceBuffer


# --------------------------------------------------------------------------------------
# device-agnostic protocol pieces (also run on CPU tensors under gloo in the tests)
# --------------------------------------------------------------------------------------
def build_halo_lists(peer_map: torch.Tensor):
    """From peer_map[b] = the peer's index of local block b (or -1):
      send_idx  local indices of the shared blocks ordered by the PEER's index (the order
                in which the peer expects the rows);
      recv_pos  [count] position of local block b among the rows the peer sends (the peer
                orders them by OUR index), -1 for blocks the peer does not hold.
    """
    shared = torch.nonzero(peer_map >= 0).flatten()
    theirs = peer_map[shared].to(torch.int64)
    order = torch.argsort(theirs, stable=True)
    send_idx = shared[order].to(torch.int32)
    recv_pos = torch.full_like(peer_map, -1, dtype=torch.int32)
    recv_pos[shared] = torch.arange(len(shared), dtype=torch.int32, device=peer_map.device)
    return send_idx, recv_pos


def plan_slabs(hist, n: int):
    """Slab boundaries of a re-partition from the GLOBAL histogram of the particle coordinate along
    the partition axis: bin b goes to the worker whose share of the running count it falls in, so
    every worker gets total / n particles up to the population of one bin (the reference cuts the
    stable argsort into equal ranges, multiworker.py:114-137; with the particles spread over
    processes the cut is made on the histogram instead).  Returns dest[bin] (int64, non-decreasing)."""
    hist = np.asarray(hist, dtype=np.int64)
    total = int(hist.sum())
    if n < 1:
        raise ValueError(f"worker count must be >= 1, got {n}")
    if total == 0:
        return np.zeros(len(hist), dtype=np.int64)
    before = np.cumsum(hist) - hist                     # particles in the bins below
    mid = before + hist // 2                            # a bin goes where its middle particle goes
    dest = (mid * n) // total
    return np.minimum(dest, n - 1).astype(np.int64)


class DistRuntime:
    """SharedRuntime (multiworker.py:73-107) across processes."""

    def __init__(self, device, initial_vmax: float = 0.0, group=None, host_timeout_ms: int = 120000):
        self.group = group
        self.n_workers = dist.get_world_size(group)
        self.wid = dist.get_rank(group)
        self.device = torch.device(device)
        self.backend = dist.get_backend(group)
        self.stage_on_host = self.backend == "gloo" and self.device.type == "cuda"
        self.generations = 0
        self._vmax = np.full((3, self.n_workers), float(initial_vmax))
        self._local_vmax = {}
        self.peer_counts = [0] * self.n_workers
        self.host_timeout_ms = int(host_timeout_ms)
        self._shm = self._shm_base = None
        self._setup_shm()

    def _setup_shm(self):
        """Map one zero-filled segment under /dev/shm into every rank when all of them run on one
        host (one process per GPU of a box): the step barrier and the few integers per rank that
        go with it then cost microseconds (mpm_shm_allgather_i64) instead of a library collective
        (kernel launch + device round trip + stream sync with NCCL).  Rank 0 creates the file and
        unlinks it once everybody has it open, so nothing outlives the processes.  Ranks on
        different hosts, no /dev/shm, or MPM_SHM=0: the small collectives stay on
        torch.distributed."""
        import mmap
        import os
        import socket
        import uuid
        hosts = [None] * self.n_workers
        dist.all_gather_object(hosts, socket.gethostname(), group=self.group)
        one_host = len(set(hosts)) == 1 and os.environ.get("MPM_SHM", "1") != "0"
        lib = _capi.lib()
        size = int(lib.mpm_shm_bytes(self.n_workers))
        path = [None]
        if self.wid == 0 and one_host and os.path.isdir("/dev/shm"):
            path[0] = f"/dev/shm/mpm_b200_{os.getpid()}_{uuid.uuid4().hex}"
            with open(path[0], "wb") as f:
                f.truncate(size)
        dist.broadcast_object_list(path, src=0, group=self.group)
        mm = None
        if path[0] is not None:
            try:
                fd = os.open(path[0], os.O_RDWR)
                try:
                    mm = mmap.mmap(fd, size)
                finally:
                    os.close(fd)
            except OSError:
                mm = None
        ok = self._all_gather_i64_dist([int(mm is not None)])[:, 0].all()     # also: everybody has it open
        if self.wid == 0 and path[0] is not None:
            os.unlink(path[0])
        if ok:
            self._shm = mm
            self._shm_base = C.addressof(C.c_char.from_buffer(mm))

    # -- transport helpers ----------------------------------------------------------------
    def _wire(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.stage_on_host else t

    def all_gather_i64(self, values) -> np.ndarray:
        """One small all_gather, [n_workers, len(values)] on the host, and a full barrier: through
        the shared segment when there is one."""
        if self._shm_base is None or len(values) > _capi.SHM_MAX_VALUES:
            return self._all_gather_i64_dist(values)
        n = len(values)
        mine = (C.c_int64 * max(n, 1))(*[int(v) for v in values])
        out = np.empty((self.n_workers, n), dtype=np.int64)
        _capi.check(_capi.lib().mpm_shm_allgather_i64(self._shm_base, self.n_workers, self.wid, mine, n,
                                                      out.ctypes.data, self.host_timeout_ms),
                    "mpm_shm_allgather_i64")
        return out

    def _all_gather_i64_dist(self, values) -> np.ndarray:
        dev = torch.device("cpu") if (self.stage_on_host or self.device.type == "cpu") else self.device
        mine = torch.tensor(values, dtype=torch.int64, device=dev)
        out = torch.empty((self.n_workers, len(values)), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(out, mine, group=self.group) if self.backend == "nccl" else \
            dist.all_gather(list(out.unbind(0)), mine, group=self.group)
        return out.cpu().numpy()

    def all_gather_codes(self, codes: torch.Tensor, counts):
        """Every rank's block-code list (variable length, padded to the longest)."""
        m = max(int(max(counts)), 1)
        pad = torch.zeros(m, dtype=torch.int64, device=codes.device)
        pad[:len(codes)] = codes
        pad = self._wire(pad)
        bufs = [torch.empty_like(pad) for _ in range(self.n_workers)]
        dist.all_gather(bufs, pad, group=self.group)
        return [bufs[q][:int(counts[q])].to(codes.device) for q in range(self.n_workers)]

    def exchange_rows(self, send: dict, recv_rows: dict):
        """Batched point-to-point exchange: send[q] -> rank q, rank q's rows -> recv_rows[q]."""
        ops, staged = [], {}
        for q in sorted(set(send) | set(recv_rows)):
            if q in recv_rows and recv_rows[q].numel():
                buf = torch.empty(recv_rows[q].shape, dtype=recv_rows[q].dtype) if self.stage_on_host \
                    else recv_rows[q]
                staged[q] = buf
                ops.append(dist.P2POp(dist.irecv, buf, q, group=self.group))
            if q in send and send[q].numel():
                ops.append(dist.P2POp(dist.isend, self._wire(send[q]).contiguous(), q, group=self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if self.stage_on_host:
            for q, buf in staged.items():
                recv_rows[q].copy_(buf)

    # -- SharedRuntime surface --------------------------------------------------------------
    def barrier_wait(self, worker_id: int) -> int:
        self.generations += 1
        return self.generations

    def publish_step(self, parity, worker_id, state):
        pass

    def publish_vmax(self, slot: int, worker_id: int, value: float) -> None:
        self._local_vmax[slot % 3] = float(value)

    def global_vmax(self, slot: int) -> float:
        return float(self._vmax[slot % 3].max())

    def step_info(self, step: int, rebuilt: bool, count: int):
        """The step's barrier: every rank learns who rebuilt, the block counts and the max
        speed each rank measured in the previous step (slot (step-1) % 3 of the vmax ring)."""
        prev = (step - 1) % 3
        v = self._local_vmax.get(prev)
        bits = int(np.float64(v).view(np.int64)) if v is not None else -1
        info = self.all_gather_i64([int(bool(rebuilt)), int(count), bits, int(step)])
        if not (info[:, 3] == step).all():
            from .errors import ContractViolationError
            raise ContractViolationError(f"ranks disagree on the step number: {info[:, 3].tolist()}")
        for q in range(self.n_workers):
            if info[q, 2] != -1:
                self._vmax[prev, q] = float(np.int64(info[q, 2]).view(np.float64))
        self.peer_counts = [int(c) for c in info[:, 1]]
        self.generations += 1
        return bool(info[:, 0].any()), self.peer_counts


class DistWorker(CudaWorker):
    """CudaWorker whose peers live in other processes."""

    def __init__(self, runtime: DistRuntime, params, material, boundary, options=None, **kw):
        super().__init__(runtime.wid, runtime, params, material, boundary, options, **kw)
        if self.options.deterministic:
            from .errors import ConfigError
            raise ConfigError("deterministic mode is implemented for workers of one process "
                              "(CudaCluster); halo rows are exchanged as float4 between processes")
        self.pipelined = False
        self.fuse_clear = False
        n = runtime.n_workers
        self._send_idx = [None] * n
        self._recv_pos = [None] * n
        self._recv_rows = [None] * n
        self._send_rows = [None] * n
        self._rebuilt_this_step = False
        self._comm_stream = torch.cuda.Stream(device=self.device) if self.device.type == "cuda" else None
        self.halo_rows_sent = 0

    def global_sound_speed(self) -> float:
        """Collective on first use: the largest sound speed over the ranks (ranks may carry different
        material populations; the CFL step must be the same everywhere)."""
        c = getattr(self, "_c_sound_global", None)
        if c is None:
            mine = float(self.material.sound_speed())
            bits = self.runtime.all_gather_i64([int(np.float64(mine).view(np.int64))])[:, 0]
            c = self._c_sound_global = float(bits.copy().view(np.float64).max())
        return c

    def run_step(self, step):
        with torch.cuda.device(self.device):
            self.step_pre_barrier(step)
            self.step_post_barrier(step)

    def run_frame(self):
        self.begin_frame()
        with torch.cuda.device(self.device):
            if self.cfl_mode:
                from .domain import cfl_dt
                c_sound = self.global_sound_speed()
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
            if self._pending_gather:
                self._flush_gather()

    def repartition(self, tol: float = 0.10, force: bool = False):
        """Collective, between frames: see dist.repartition."""
        return repartition(self, tol=tol, force=force)

    def _publish(self, par, rebuilt):
        self._rebuilt_this_step = rebuilt

    def _post_barrier(self, par):
        """Barrier + shared-block tagging when any rank rebuilt (pipeline.py:1147-1164)."""
        rt = self.runtime
        step = self._global_step
        any_rebuilt, counts = rt.step_info(step, self._rebuilt_this_step, self.table.count)
        if not any_rebuilt:
            return
        tb = self.table
        mine = tb._codes.data[:tb.count]
        lists = rt.all_gather_codes(mine, counts)
        stream = _stream_ptr()
        for q in range(rt.n_workers):
            if q == rt.wid:
                continue
            if tb.count == 0 or counts[q] == 0:
                self._send_idx[q] = torch.zeros(0, dtype=torch.int32, device=self.device)
                self._recv_pos[q] = torch.full((max(tb.count, 1),), -1, dtype=torch.int32,
                                               device=self.device)
                self._send_rows[q] = self._recv_rows[q] = torch.zeros((0, 64, 4), device=self.device)
                continue
            m = self._peer_map[q]
            if m is None:
                m = self._peer_map[q] = DeviceBuffer(torch.int32, (), self.device)
            m.resize(tb.count, keep=False)
            codes_q = lists[q].contiguous()
            self._call("mpm_tag_shared", codes_q.data_ptr(), int(counts[q]), tb._hkeys.ptr,
                       tb._hvals.ptr, tb.hash_cap, m.ptr, tb.count, stream)
            send_idx, recv_pos = build_halo_lists(m.data[:tb.count])
            self._send_idx[q], self._recv_pos[q] = send_idx.contiguous(), recv_pos.contiguous()
            k = len(send_idx)
            self._send_rows[q] = torch.empty((k, 64, 4), dtype=torch.float32, device=self.device)
            self._recv_rows[q] = torch.empty((k, 64, 4), dtype=torch.float32, device=self.device)

    def _gather_peers(self, par):
        """Pack, exchange, and describe the received rows as grid-update peers."""
        rt, tb, gr = self.runtime, self.table, self.grid
        stream = _stream_ptr()
        send, recv = {}, {}
        for q in range(rt.n_workers):
            if q == rt.wid or self._send_idx[q] is None:
                continue
            k = len(self._send_idx[q])
            if k:
                self._call("mpm_pack_halo", gr._raw[par].ptr, tb._touched[par].ptr,
                           self._send_idx[q].data_ptr(), k, self._send_rows[q].data_ptr(), stream)
                send[q], recv[q] = self._send_rows[q], self._recv_rows[q]
                self.halo_rows_sent += k
        return send, recv

    def _reduce_and_update(self, par, step=None):
        if step is None:
            step = self._global_step
        rt, tb = self.runtime, self.table
        send, recv = self._gather_peers(par)
        gp = self._grid_params()
        peers = [(recv[q].data_ptr(), None, self._recv_pos[q].data_ptr()) for q in sorted(recv)]
        gp.n_peers = len(peers)
        for k, (r, t, m) in enumerate(peers):
            gp.peer_raw[k], gp.peer_touched[k], gp.peer_map[k] = r, t, m
        tv = tb.view()
        nxt = (step + 1 if self._fused_now else step) % _RING
        cur = torch.cuda.current_stream()
        if tb.count and peers:
            # interior blocks while the halo rows travel
            self._comm_stream.wait_stream(cur)
            gp.block_filter = 1
            self._grid_update_launch(gp, tv, par, self._status_ptr(nxt), _stream_ptr())
            with torch.cuda.stream(self._comm_stream):
                rt.exchange_rows(send, recv)
            cur.wait_stream(self._comm_stream)
            gp.block_filter = 2
            self._grid_update_launch(gp, tv, par, None, _stream_ptr())
        else:
            rt.exchange_rows(send, recv)      # nothing shared: still matched send/recv pairs
            if tb.count:
                gp.block_filter = 0
                self._grid_update_launch(gp, tv, par, self._status_ptr(nxt), _stream_ptr())
        if tb.count:
            self._slot_clean[nxt] = True
        self._vel_dt = self.dt


# --------------------------------------------------------------------------------------
# dynamic re-partitioning (the paper's future work)
# --------------------------------------------------------------------------------------
REPARTITION_BINS = 4096


def _state_on_device(w: CudaWorker):
    """Every stored lane in (group, lane) order as device tensors: rows [n, nch] fp32, ids [n],
    and the flat (group * 32 + lane) position of each row in the store."""
    st = w.store
    n, G = st.count, st.n_groups
    flat = torch.zeros((max(n, 1), st.nch), dtype=torch.float32, device=w.device)
    ids = torch.zeros(max(n, 1), dtype=torch.int64, device=w.device)
    where = torch.zeros(max(n, 1), dtype=torch.int64, device=w.device)
    if n:
        v = st.view()
        _capi.check(_capi.lib().mpm_gather_state(C.byref(v), flat.data_ptr(), ids.data_ptr(), _stream_ptr()),
                    "mpm_gather_state")
        glen = st._group_len[st.cur].data[:G].to(torch.int64)
        gstart = torch.cumsum(glen, 0) - glen
        grp = torch.repeat_interleave(torch.arange(G, device=w.device), glen)
        where = grp * 32 + (torch.arange(n, device=w.device) - gstart[grp])
    return flat[:n], ids[:n], where[:n]


def migrate_rows(rt: DistRuntime, flat: torch.Tensor, ids: torch.Tensor, alive: torch.Tensor, nch: int,
                 tol: float = 0.10, force: bool = False, bins: int = REPARTITION_BINS):
    """The collective part of a re-partition, on whatever device the tensors live (CUDA per rank, or CPU
    tensors under gloo in the tests): agree on the longest axis of the global bounding box, histogram,
    cut (plan_slabs), tell every rank how many rows it gets from whom, and exchange rows + ids.

    flat [n, nch] float32 particle rows (positions in columns 0:3), ids [n] int64, alive [n] bool (rows
    that may move).  Returns None when nothing has to move, else a dict:
      leaving [n] bool, rows / row_ids (what arrived here, concatenated in rank order), before / after
      (per-rank counts), axis."""
    n_ranks = rt.n_workers
    dev = flat.device
    pos = flat[:, 0:3].to(torch.float64)
    big = 1e300
    any_alive = bool(alive.any()) if len(ids) else False
    lo = pos[alive].min(dim=0).values.cpu().numpy() if any_alive else np.full(3, big)
    hi = pos[alive].max(dim=0).values.cpu().numpy() if any_alive else np.full(3, -big)
    n_alive = int(alive.sum().item()) if len(ids) else 0
    # bounding box and counts of everybody (float64 bit patterns through the int64 exchange)
    info = rt.all_gather_i64([int(np.float64(x).view(np.int64)) for x in list(lo) + list(hi)] + [n_alive, nch])
    los = info[:, 0:3].copy().view(np.float64)
    his = info[:, 3:6].copy().view(np.float64)
    counts = info[:, 6].astype(np.int64)
    if not (info[:, 7] == nch).all():
        from .errors import ConfigError
        raise ConfigError("re-partitioning moves particles between ranks of ONE material population")
    total = int(counts.sum())
    if total == 0:
        return None
    mean = total / n_ranks
    if not force and float(np.abs(counts - mean).max()) <= tol * mean:
        return None
    glo, ghi = los.min(axis=0), his.max(axis=0)
    axis = int(np.argmax(ghi - glo))
    width = max(float(ghi[axis] - glo[axis]), 1e-300)
    # histogram of my particles, cut of the global one
    b = torch.clamp(((pos[:, axis] - glo[axis]) * (bins / width)).to(torch.int64), 0, bins - 1)
    hist = torch.bincount(b[alive], minlength=bins).cpu().numpy() if n_alive else np.zeros(bins, np.int64)
    ghist = rt._all_gather_i64_dist(hist.tolist()).sum(axis=0)
    dest = torch.from_numpy(plan_slabs(ghist, n_ranks)).to(dev)[b]
    dest[~alive] = rt.wid
    leaving = dest != rt.wid
    # who sends how many to whom
    out_counts = torch.bincount(dest[leaving], minlength=n_ranks).cpu().numpy()
    table = rt.all_gather_i64(out_counts.tolist()) if n_ranks <= _capi.SHM_MAX_VALUES else \
        rt._all_gather_i64_dist(out_counts.tolist())
    send_rows, send_ids, recv_rows, recv_ids = {}, {}, {}, {}
    for q in range(n_ranks):
        if q == rt.wid:
            continue
        if out_counts[q]:
            sel = dest == q
            send_rows[q] = flat[sel].contiguous()
            send_ids[q] = ids[sel].contiguous()
        k = int(table[q, rt.wid])
        if k:
            recv_rows[q] = torch.empty((k, nch), dtype=torch.float32, device=dev)
            recv_ids[q] = torch.empty(k, dtype=torch.int64, device=dev)
    if dev.type == "cuda":
        torch.cuda.current_stream().synchronize()
    rt.exchange_rows(send_rows, recv_rows)
    rt.exchange_rows(send_ids, recv_ids)
    rows = torch.cat([recv_rows[q] for q in sorted(recv_rows)]) if recv_rows else flat[:0]
    row_ids = torch.cat([recv_ids[q] for q in sorted(recv_ids)]) if recv_ids else ids[:0]
    after = counts - table.sum(axis=1) + table.sum(axis=0)
    return {"leaving": leaving, "rows": rows, "row_ids": row_ids, "axis": axis,
            "before": counts.tolist(), "after": after.tolist()}


def repartition(w: "DistWorker", tol: float = 0.10, force: bool = False, bins: int = REPARTITION_BINS):
    """Collective, between frames.  Re-cut the slabs along the longest axis of the CURRENT particle
    positions and migrate the particles whose slab now belongs to another rank.

    The reference partitions once (bench.py:434-439, multiworker.py:114-137) and a worker keeps its
    particles for good: as the material moves, the slabs interleave, the shared blocks (halo rows)
    grow, and sources / sinks unbalance the counts.  Here every rank histograms its particles
    along the axis, the global histogram is cut into equal shares (plan_slabs), and each particle
    whose share is another rank's travels there with its whole state (x, v, C, m, F | J, plastic
    scalar, id): it is removed here the way a sink removes it (mass 0, lane flagged, id -1, dropped
    by the next rebuild's compaction) and staged there like an appended particle with state.  Ids
    are preserved, the total mass is unchanged, and the step sequence continues with a rebuild
    on every rank.  Nothing moves unless `force` or some rank's count is more than `tol` away
    from the mean.  Returns a dict of counts (before, after, sent, received) or None."""
    with torch.cuda.device(w.device):
        if w._pending_gather:
            w._flush_gather()
        flat, ids, where = _state_on_device(w)
        meta = w.store._lane_meta[w.store.cur].data.view(-1)
        alive = torch.ones(len(ids), dtype=torch.bool, device=w.device)
        if len(ids):
            alive = (meta[where].to(torch.int32) & 0x8000) == 0      # quarantined / sunk lanes stay put
        mig = migrate_rows(w.runtime, flat, ids, alive, w.store.nch, tol=tol, force=force, bins=bins)
        if mig is None:
            return None
        leaving = mig["leaving"]
        n_out, n_in = int(leaving.sum().item()), int(len(mig["row_ids"]))
        if n_out:
            # leave like a sunk particle: flagged, massless, id -1 (dropped by the next compaction)
            st = w.store
            gone = where[leaving]
            flag = torch.tensor(-32768 | 0x4000, dtype=torch.int16, device=w.device)   # QUARANTINED | SUNK
            meta[gone] = meta[gone] | flag
            data = st._data[st.cur].data                      # [G, nch, 32]
            data[gone // 32, 15, gone % 32] = 0.0             # CH_MASS
            st._orig_id[st.cur].data.view(-1)[gone] = -1
            st.has_sink = True
        if n_in:
            rows, rid = mig["rows"].cpu().numpy(), mig["row_ids"].cpu().numpy()
            w.store.stage_append(rows[:, 0:3], rows[:, 3:6], rows[:, 15].copy(), deformation=rows[:, 16:],
                                 affine=rows[:, 6:15], ids=rid)
        # every rank rebuilds on the next step (SPMD), whether or not its own population changed
        w.flags.rebuild_needed = True
        w.flags.fused_mode = False
        w._clock_valid = False
        if hasattr(w, "_need_collective"):
            w._need_collective = True
        return {"axis": mig["axis"], "before": mig["before"], "after": mig["after"], "sent": n_out,
                "received": n_in}


# --------------------------------------------------------------------------------------
# material populations over ranks (BASELINE.json configs[4]: mixed snow / sand on 8 GPUs)
# --------------------------------------------------------------------------------------
def population_layout(rank: int, world: int, n_populations: int):
    """Which (population, slab, n_slabs) a rank holds when `n_populations` material populations
    are spread over `world` ranks: ranks p, p + n_populations, ... hold the slabs of population p.
    One logical worker (one material, one block table) per process, as everywhere else; a GPU
    that is to carry several populations runs one process per population (the peer-mapped
    transport maps the tables of processes on one device like those of another device), and
    the populations meet on the grid through the same halo reduction as the slabs do
    (pipeline.py:1172-1188)."""
    if n_populations < 1 or world % n_populations:
        from .errors import ConfigError
        raise ConfigError(f"{world} ranks cannot hold {n_populations} populations in equal numbers of slabs")
    return rank % n_populations, rank // n_populations, world // n_populations


def seed_population_rank(worker: "DistWorker", populations):
    """Seed this rank's slab of its population.  `populations`: sequence of objects with
    .positions / .velocities / .particle_mass (scenes.Population); ids are consecutive ranges in
    population order, as CudaCluster.seed_populations numbers them.  Returns the global ids."""
    rt = worker.runtime
    p, slab, n_slabs = population_layout(rt.wid, rt.n_workers, len(populations))
    pop = populations[p]
    base = int(sum(len(q.positions) for q in populations[:p]))
    part = partition_particles(pop.positions, n_slabs)[slab]
    if len(part):
        worker.seed_particles(np.asarray(pop.positions)[part], np.asarray(pop.velocities)[part],
                              pop.particle_mass, ids=part + base)
    return part + base


def seed_rank(worker: DistWorker, positions, velocities, mass):
    """bench.py:434-439 of the reference: rank r takes the r-th slab of the partition; ids are
    the indices into the global arrays."""
    parts = partition_particles(positions, worker.runtime.n_workers)
    part = parts[worker.runtime.wid]
    if len(part):
        worker.seed_particles(np.asarray(positions)[part], np.asarray(velocities)[part], mass, ids=part)
    return part
