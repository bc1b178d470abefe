"""CPU oracle: restatement of the reference `mpmbench` substep loop (float64).

THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import it.  The product
package never imports anything from oracle/.

Parity status: PINNED -- tests/test_oracle_golden.py compares every stage against
arrays dumped from the reference itself (tests/golden/make_golden.py) and against the
reference tests' known-answer vectors.

The arithmetic lives in mpm_oracle.c (built by oracle/build.py into
oracle/libmpm_oracle.so); this module restates the host-side orchestration:
  OracleWorker.run_step     <- Worker.run_step            pipeline.py:905-940
  OracleWorker._rebuild     <- Worker._rebuild            pipeline.py:958-1015
                               BlockTable.rebuild         grid.py:348-386
                               ParticleStore.histogram_sort particles.py:360-401
  OracleWorker._clear       <- Worker._clear              pipeline.py:1022-1037
  OracleWorker._reduce_and_update <- pipeline.py:1166-1231
  OracleRuntime             <- SharedRuntime              multiworker.py:73-107
  partition_particles       <- multiworker.py:114-137
  OracleCluster             <- bench._Orchestra + SpinBarrier, run in lockstep phases
                               (pre-barrier phase of every worker, then post-barrier
                               phase of every worker) which is equivalent to the
                               threaded schedule because pre-barrier work touches only
                               worker-local state.
Parameter objects are duck-typed (params.dx, material.kind, ...), so tests can pass
the product package's own SimParams/Material/BoundaryBox/PipelineOptions.
Only the default ablation arms are restated (rebuild amortized|every_step, sort
amortized|none_between, fusion merged, transfer split|g2p2g, deterministic on/off).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmpm_oracle.so")

CELL_BIAS = 64
COORD_MAX = 1 << 21
CH_POS, CH_VEL, CH_C, CH_MASS, CH_DEF = 0, 3, 6, 15, 16
N_COUNTERS = 6
C_ACCUM, C_QUARANTINE, C_DEGENERATE, C_SVD_CLAMP, C_ADDRESS_ERR, C_SUBGROUPS = range(6)
MASS_SCALE = float(2 ** 40)
MOM_SCALE = float(2 ** 32)
FREE_ZONE_LO_CELLS = 3.5
FREE_ZONE_HI_CELLS = 6.5
FUSED_MARGIN_CELLS = 1.0


class OracleSpatialDomainError(ValueError):
    pass


class OracleContractViolation(RuntimeError):
    pass


class _TransferParams(C.Structure):
    _fields_ = [("lane_width", C.c_int64), ("nch", C.c_int64), ("mat_kind", C.c_int64),
                ("mu", C.c_double), ("lam", C.c_double), ("kappa", C.c_double),
                ("gamma", C.c_double), ("clamp_tension", C.c_int64),
                ("density", C.c_double), ("dx", C.c_double),
                ("det", C.c_int64), ("do_lane_sort", C.c_int64),
                ("theta_c", C.c_double), ("theta_s", C.c_double), ("hardening", C.c_double),
                ("sand_alpha", C.c_double),
                ("sink_enabled", C.c_int64), ("sink_lo", C.c_double * 3), ("sink_hi", C.c_double * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            from . import build as _b  # type: ignore
            _b.build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_encode_cell.restype = C.c_int64
        _lib.orc_encode_cell.argtypes = [C.c_int64] * 3
        _lib.orc_particle_codes.restype = C.c_int64
        _lib.orc_dilate_and_link.restype = C.c_int64
        _lib.orc_build_groups.restype = C.c_int64
        _lib.orc_gather_live.restype = C.c_int64
        _lib.orc_corotated_tau.restype = C.c_int
        _lib.orc_fluid_tau.restype = C.c_double
        _lib.orc_fluid_tau.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _i(v):
    return C.c_int64(int(v))


def _d(v):
    return C.c_double(float(v))


# --------------------------------------------------------------------------------------
# leaf functions (thin wrappers, used directly by the golden/KAT tests)
# --------------------------------------------------------------------------------------

def encode(x, y, z):
    return int(lib().orc_encode_cell(int(x), int(y), int(z)))


def decode(code):
    out = np.zeros(3, dtype=np.int64)
    lib().orc_decode_cell(_i(code), _p(out))
    return tuple(int(v) for v in out)


def decode_batch(codes):
    codes = np.asarray(codes, dtype=np.int64)
    out = np.empty((len(codes), 3), dtype=np.int64)
    for i, c in enumerate(codes):
        out[i] = decode(int(c))
    return out


def particle_code_batch(pos, dx, bias=CELL_BIAS):
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    codes = np.empty(len(pos), dtype=np.int64)
    bad = lib().orc_particle_codes(_p(pos), _i(len(pos)), _d(dx), _i(bias), _p(codes))
    if bad >= 0:
        raise OracleSpatialDomainError(
            f"position {tuple(float(v) for v in pos[bad])} maps outside the biased domain")
    return codes


def stable_counting_sort(keys, domain=None):
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    if domain is None:
        domain = int(keys.max()) + 1 if len(keys) else 1
    counts = np.zeros(domain, dtype=np.int64)
    perm = np.empty(len(keys), dtype=np.int64)
    lib().orc_counting_sort_perm(_p(keys), _i(len(keys)), _p(counts), _i(domain), _p(perm))
    return perm


def lane_radix_sort10(keys):
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    order = np.empty(len(keys), dtype=np.int64)
    scratch = np.empty(len(keys), dtype=np.int64)
    lib().orc_radix10_order(_p(keys), _i(len(keys)), _p(order), _p(scratch))
    return order


def svd3(F):
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(9)
    u, s, v = np.empty(9), np.empty(3), np.empty(9)
    lib().orc_svd3(_p(F), _p(u), _p(s), _p(v))
    return u.reshape(3, 3), s, v.reshape(3, 3)


def corotated_tau(F, mu, lam):
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(9)
    t = np.empty(9)
    clamped = lib().orc_corotated_tau(_p(F), _d(mu), _d(lam), _p(t))
    return t.reshape(3, 3), bool(clamped)


def snow_project(F, Jp, theta_c, theta_s):
    """Return mapping of the snow model (orc_snow_project): projected F_E and updated J_P."""
    F = np.array(F, dtype=np.float64).reshape(9)
    jp = C.c_double(float(Jp))
    lib().orc_snow_project(_p(F), C.byref(jp), _d(theta_c), _d(theta_s))
    return F.reshape(3, 3), float(jp.value)


def snow_tau(FE, Jp, mu, lam, hardening):
    """Stress of a projected snow state as scatter_prep evaluates it: fixed-corotated with
    moduli hardened by exp(xi (1 - J_P))."""
    h = float(np.exp(hardening * (1.0 - Jp)))
    return corotated_tau(FE, mu * h, lam * h)[0]


def sand_project(F, vc, mu, lam, alpha):
    """Drucker-Prager return mapping (orc_sand_project): projected F_E, volume-correction scalar."""
    F = np.array(F, dtype=np.float64).reshape(9)
    v = C.c_double(float(vc))
    lib().orc_sand_project(_p(F), C.byref(v), _d(mu), _d(lam), _d(alpha))
    return F.reshape(3, 3), float(v.value)


def sand_tau(F, mu, lam):
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(9)
    t = np.empty(9)
    lib().orc_sand_tau(_p(F), _d(mu), _d(lam), _p(t))
    return t.reshape(3, 3)


def fluid_tau(J, kappa, gamma, clamp_tension=False):
    return float(lib().orc_fluid_tau(float(J), float(kappa), float(gamma), int(bool(clamp_tension))))


def quadratic_weights(position, dx):
    """domain.py:150-164 (host helper; uses division like the reference)."""
    pos = np.asarray(position, dtype=np.float64)
    base = np.floor(pos / dx - 0.5).astype(np.int64)
    f = pos / dx - base
    w = np.stack([0.5 * (1.5 - f) ** 2, 0.75 - (f - 1.0) ** 2, 0.5 * (f - 0.5) ** 2], axis=-1)
    return base, w


def cfl_dt(max_speed, params, frame_remaining):
    """domain.py:523-532"""
    dt = params.cfl * params.dx / max(max_speed, 1e-12)
    return min(frame_remaining, dt)


def sound_speed(material):
    """domain.py:95-100"""
    if int(material.kind) == 0:
        return float(np.sqrt(material.gamma * material.bulk_modulus / material.density))
    return float(np.sqrt((material.lam + 2.0 * material.mu) / material.density))


def partition_particles(positions, n):
    """multiworker.py:114-137"""
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


# --------------------------------------------------------------------------------------
# hash + block table: grid.py:176-257, 325-386
# --------------------------------------------------------------------------------------

class OracleHash:
    def __init__(self):
        self._alloc(1024)
        self.count = 0

    def _alloc(self, cap):
        self.capacity = cap
        self.shift = 64 - cap.bit_length() + 1
        self.mask = cap - 1
        self.keys = np.full(cap, -1, dtype=np.int64)
        self.vals = np.full(cap, -1, dtype=np.int64)

    def clear(self):
        self.keys.fill(-1)
        self.vals.fill(-1)
        self.count = 0

    def ensure_room(self, extra):
        needed = 2 * (self.count + extra)  # load factor < 0.5 (grid.py:214-229)
        if needed <= self.capacity // 2:
            return
        cap = 1 << (int(4 * needed) - 1).bit_length()
        live = self.keys != -1
        codes, idx = self.keys[live], self.vals[live]
        self._alloc(cap)
        # reinsert preserving indices (grid.py:260-268); order is irrelevant to results
        for c, i in zip(codes, idx):
            j = self._slot(int(c))
            while self.keys[j] != -1:
                j = (j + 1) & self.mask
            self.keys[j] = c
            self.vals[j] = i

    def _slot(self, key):
        prod = (key * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        if prod >= 1 << 63:
            prod -= 1 << 64
        return (prod >> self.shift) & self.mask

    def insert_batch(self, codes):
        codes = np.ascontiguousarray(codes, dtype=np.int64)
        self.ensure_room(len(codes))
        out = np.empty(len(codes), dtype=np.int64)
        box = np.array([self.count], dtype=np.int64)
        lib().orc_hash_insert_batch(_p(self.keys), _p(self.vals), _i(self.shift), _i(self.mask),
                                    _p(codes), _i(len(codes)), _p(out), _p(box))
        self.count = int(box[0])
        return out

    def lookup_batch(self, codes):
        codes = np.ascontiguousarray(codes, dtype=np.int64)
        out = np.empty(len(codes), dtype=np.int64)
        lib().orc_hash_lookup_batch(_p(self.keys), _p(self.vals), _i(self.shift), _i(self.mask),
                                    _p(codes), _i(len(codes)), _p(out))
        return out


class OracleTable:
    """BlockTable: grid.py:325-401"""

    def __init__(self):
        self.hash = OracleHash()
        self.codes = np.zeros(0, dtype=np.int64)
        self.neighbor = np.zeros((1, 27), dtype=np.int32)
        self.touched = [np.zeros(0, dtype=np.uint8), np.zeros(0, dtype=np.uint8)]
        self.count = 0
        self.n_gblocks = 0

    def rebuild(self, gblock_codes):
        self.hash.clear()
        codes = np.ascontiguousarray(gblock_codes, dtype=np.int64)
        gidx = self.hash.insert_batch(codes)
        n_g = self.hash.count
        upper = n_g * 27
        dense = np.zeros(max(upper, 1), dtype=np.int64)
        self.neighbor = np.zeros((max(n_g, 1), 27), dtype=np.int32)
        uniq = np.empty(n_g, dtype=np.int64)
        uniq[gidx] = codes
        dense[:n_g] = uniq
        self.hash.ensure_room(upper - n_g)
        box = np.array([n_g], dtype=np.int64)
        bad = lib().orc_dilate_and_link(_p(self.hash.keys), _p(self.hash.vals),
                                        _i(self.hash.shift), _i(self.hash.mask), _p(box),
                                        _p(uniq), _i(n_g), _p(dense), _p(self.neighbor))
        if bad >= 0:
            x, y, z = decode(int(uniq[bad]))
            raise OracleSpatialDomainError(
                f"block ({x - CELL_BIAS // 4}, {y - CELL_BIAS // 4}, {z - CELL_BIAS // 4}) "
                f"touches the domain boundary; scenes must leave a one-block margin")
        self.hash.count = int(box[0])
        self.count = int(box[0])
        self.n_gblocks = int(n_g)
        self.codes = dense[:self.count].copy()
        for k in (0, 1):
            old = self.touched[k]
            new = np.zeros(self.count, dtype=np.uint8)
            m = min(len(old), self.count)
            new[:m] = old[:m]   # GrowBuffer.resize keeps old contents (memory.py:48-69)
            self.touched[k] = new
        return gidx

    def touched_indices(self, buffer=0):
        return np.flatnonzero(self.touched[buffer][:self.count])


# --------------------------------------------------------------------------------------
# particle store: particles.py:268-487
# --------------------------------------------------------------------------------------

class OracleStore:
    def __init__(self, kind, lane_width=32):
        self.kind = int(kind)
        self.lane_width = int(lane_width)
        # kinds 2/3 (snow, sand: not in the reference) carry one plastic scalar in channel 25
        self.nch = 17 if self.kind == 0 else (25 if self.kind == 1 else 26)
        LW = self.lane_width
        self.data = np.zeros((1, self.nch, LW))
        self.orig_id = np.zeros((1, LW), dtype=np.int64)
        self.lane_key = np.zeros((1, LW), dtype=np.int64)
        self.quarantined = np.zeros((1, LW), dtype=np.uint8)
        self.group_len = np.zeros(0, dtype=np.int32)
        self.group_block = np.zeros(0, dtype=np.int32)
        self.group_origin = np.zeros((1, 3), dtype=np.int32)
        self.n_groups = 0
        self.count = 0
        self._staged = []
        self.staged_count = 0
        self._next_id = 0

    def default_deformation(self, n):
        if self.kind == 0:
            return np.ones((n, 1))
        return np.tile(np.eye(3).reshape(9), (n, 1))

    def stage_append(self, positions, velocities, masses, deformation=None, affine=None, ids=None):
        pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
        n = pos.shape[0]
        if n == 0:
            return 0
        vel = np.atleast_2d(np.asarray(velocities, dtype=np.float64))
        mass = np.broadcast_to(np.asarray(masses, dtype=np.float64), (n,)).copy()
        defo = self.default_deformation(n) if deformation is None \
            else np.asarray(deformation, dtype=np.float64).reshape(n, -1)
        Cm = np.zeros((n, 9)) if affine is None else np.asarray(affine, dtype=np.float64).reshape(n, 9)
        if ids is None:
            ids = np.arange(self._next_id, self._next_id + n, dtype=np.int64)
            self._next_id += n
        else:
            ids = np.asarray(ids, dtype=np.int64).reshape(n)
            self._next_id = max(self._next_id, int(ids.max()) + 1)
        self._staged.append((pos, vel, Cm, mass, defo, ids))
        self.staged_count += n
        return n

    def _gather_live(self, include_quarantined=False):
        total = max(self.count, 1)
        flat = np.zeros((total, self.nch))
        ids = np.empty(total, dtype=np.int64)
        n = 0
        if self.n_groups:
            q = None if include_quarantined else self.quarantined
            n = lib().orc_gather_live(_p(self.data), _i(self.n_groups), _i(self.nch),
                                      _i(self.lane_width), _p(self.group_len), _p(q),
                                      _p(self.orig_id), _p(flat), _p(ids))
        return flat[:n], ids[:n]

    def gather_flat(self):
        live, lids = self._gather_live()
        total = len(lids) + self.staged_count
        flat = np.zeros((total, self.nch))
        ids = np.empty(total, dtype=np.int64)
        n = len(lids)
        flat[:n] = live
        ids[:n] = lids
        for pos, vel, Cm, mass, defo, sid in self._staged:
            m = pos.shape[0]
            flat[n:n + m, CH_POS:CH_POS + 3] = pos
            flat[n:n + m, CH_VEL:CH_VEL + 3] = vel
            flat[n:n + m, CH_C:CH_C + 9] = Cm
            flat[n:n + m, CH_MASS] = mass
            flat[n:n + m, CH_DEF:CH_DEF + defo.shape[1]] = defo
            if self.nch > 25 and defo.shape[1] <= 9:
                flat[n:n + m, 25] = 1.0 if self.kind == 2 else 0.0
            ids[n:n + m] = sid
            n += m
        self._staged.clear()
        self.staged_count = 0
        return flat[:n], ids[:n]

    def histogram_sort(self, flat, ids, keys):
        n = len(keys)
        LW = self.lane_width
        domain = ((int(keys.max()) >> 6) + 1) << 6 if n else 1
        counts = np.zeros(domain, dtype=np.int64)
        perm = np.empty(n, dtype=np.int64)
        keys = np.ascontiguousarray(keys, dtype=np.int64)
        lib().orc_counting_sort_perm(_p(keys), _i(n), _p(counts), _i(domain), _p(perm))
        sorted_block = np.ascontiguousarray(keys[perm] >> 6, dtype=np.int64)
        self.group_len = np.zeros(n + 1, dtype=np.int32)
        self.group_block = np.zeros(n + 1, dtype=np.int32)
        slot_group = np.empty(n, dtype=np.int64)
        slot_lane = np.empty(n, dtype=np.int64)
        ng = int(lib().orc_build_groups(_p(sorted_block), _i(n), _i(LW), _p(self.group_len),
                                        _p(self.group_block), _p(slot_group), _p(slot_lane))) if n else 0
        self.n_groups = ng
        self.group_len = self.group_len[:ng].copy()
        self.group_block = self.group_block[:ng].copy()
        self.group_origin = np.zeros((max(ng, 1), 3), dtype=np.int32)
        self.data = np.zeros((max(ng, 1), self.nch, LW))
        self.orig_id = np.zeros((max(ng, 1), LW), dtype=np.int64)
        self.lane_key = np.zeros((max(ng, 1), LW), dtype=np.int64)
        self.quarantined = np.zeros((max(ng, 1), LW), dtype=np.uint8)
        if n:
            flat = np.ascontiguousarray(flat)
            ids = np.ascontiguousarray(ids)
            lib().orc_scatter_sorted(_p(flat), _p(ids), _p(perm), _i(n), _i(self.nch), _i(LW),
                                     _p(slot_group), _p(slot_lane), _p(self.data), _p(self.orig_id))
        self.count = n
        return perm

    def refresh_lane_keys(self, dx, bias=CELL_BIAS):
        if self.n_groups:
            lib().orc_recompute_lane_keys(_p(self.data), _i(self.n_groups), _i(self.nch),
                                          _i(self.lane_width), _p(self.group_len),
                                          _p(self.group_origin), _d(1.0 / dx), _i(bias),
                                          _p(self.lane_key))

    def positions_with_ids(self):
        flat, ids = self.state_with_ids()
        return flat[:, CH_POS:CH_POS + 3].copy(), ids.copy()

    def state_with_ids(self):
        """All channels of stored particles (incl. quarantined) + ids; oracle-only helper.
        Lanes emptied by a particle sink (id -1) are skipped."""
        flat, ids = self._gather_live(include_quarantined=True)
        keep = ids >= 0
        return (flat, ids) if keep.all() else (flat[keep], ids[keep])

    def total_mass(self):
        return float(self.data[:self.n_groups, CH_MASS, :].sum()) if self.n_groups else 0.0

    def total_momentum(self):
        if not self.n_groups:
            return np.zeros(3)
        d = self.data[:self.n_groups]
        m = d[:, CH_MASS, :]
        return np.array([(m * d[:, CH_VEL + a, :]).sum() for a in range(3)])


class OracleGrid:
    def __init__(self):
        self.raw = [np.zeros((0, 4, 64)), np.zeros((0, 4, 64))]
        self.vel = np.zeros((0, 4, 64))
        self.vel_old = None
        self.count = 0


# --------------------------------------------------------------------------------------
# runtime + worker
# --------------------------------------------------------------------------------------

class OracleRuntime:
    """SharedRuntime minus the barrier (OracleCluster runs the phases in lockstep)."""

    def __init__(self, n_workers, initial_vmax=0.0):
        self.n_workers = n_workers
        self._steps = [[None] * n_workers, [None] * n_workers]
        self._vmax = np.full((3, n_workers), float(initial_vmax))
        self.generations = 0

    def publish_step(self, parity, wid, state):
        self._steps[parity & 1][wid] = state

    def peer_step(self, parity, wid):
        return self._steps[parity & 1][wid]

    def publish_vmax(self, slot, wid, value):
        self._vmax[slot % 3, wid] = value

    def global_vmax(self, slot):
        return float(self._vmax[slot % 3].max())


class _Opts:
    rebuild = "amortized"
    sort = "amortized"
    fusion = "merged"
    transfer = "split"
    deterministic = False
    fused_threshold = 100_000
    collect_conservation = False


def _resize_rows(arr, count):
    """GrowBuffer.resize semantics for the live region: keep old rows, new rows zero."""
    if arr.shape[0] == count:
        return arr
    out = np.zeros((count,) + arr.shape[1:], dtype=arr.dtype)
    m = min(arr.shape[0], count)
    out[:m] = arr[:m]
    return out


class OracleWorker:
    def __init__(self, wid, runtime, params, material, boundary, options=None):
        self.wid = wid
        self.runtime = runtime
        self.params = params
        self.material = material
        self.boundary = boundary
        self.options = options if options is not None else _Opts()
        self.store = OracleStore(int(material.kind), params.lane_width)
        self.table = OracleTable()
        self.grid = OracleGrid()
        self.rebuild_needed = True
        self.steps_since_rebuild = 0
        self.fused_mode = False
        self.counters = np.zeros(N_COUNTERS, dtype=np.int64)
        self.conservation = []
        self.rebuild_steps = []
        self.dt = params.dt
        self._vel_dt = params.dt
        self._global_step = 0
        self._pending_gather = False
        self._pending_full_clear_parity = -1
        self._published_codes = (np.zeros(0, dtype=np.int64), 0)
        self._peer_map = [None] * runtime.n_workers
        self._peer_states = None
        self.cfl_mode = False
        self.frame_steps = 0
        self.last_perm = None
        self.last_gidx = None
        m = material
        self._tp = _TransferParams(
            lane_width=params.lane_width, nch=self.store.nch, mat_kind=int(m.kind),
            mu=float(m.mu), lam=float(m.lam), kappa=float(m.bulk_modulus), gamma=float(m.gamma),
            clamp_tension=int(bool(m.clamp_tension)), density=float(m.density),
            dx=float(params.dx), det=int(bool(self.options.deterministic)),
            do_lane_sort=int(self.options.sort != "none_between"),
            theta_c=float(getattr(m, "theta_c", 0.0)), theta_s=float(getattr(m, "theta_s", 0.0)),
            hardening=float(getattr(m, "hardening", 0.0)),
            sand_alpha=math.sqrt(2.0 / 3.0) * 2.0 * math.sin(math.radians(getattr(m, "friction_angle", 30.0)))
            / (3.0 - math.sin(math.radians(getattr(m, "friction_angle", 30.0)))))

    # -- particle sink (not in the reference; mirrors CudaWorker.set_sink) --
    def set_sink(self, min_corner, max_corner):
        self._tp.sink_enabled = 1
        for k in range(3):
            self._tp.sink_lo[k], self._tp.sink_hi[k] = float(min_corner[k]), float(max_corner[k])
        self.removed_count = getattr(self, "removed_count", 0)
        self._sunk_pending = False

    def _after_gather_stats(self, stats):
        if stats[2] > 0.0:
            self.removed_count += int(stats[2])
            self._sunk_pending = True
            self.store.orig_id[:self.store.n_groups][self.store.quarantined[:self.store.n_groups] == 2] = -1

    # -- population --
    def seed_particles(self, positions, velocities, masses, ids):
        n = self.store.stage_append(positions, velocities, masses, ids=ids)
        self.rebuild_needed = True
        return n

    def append_particles(self, positions, velocities, masses, ids=None):
        if len(np.atleast_2d(positions)) == 0:
            return 0
        if self.fused_mode:
            raise OracleContractViolation("cannot add particles while fused")
        n = self.store.stage_append(positions, velocities, masses, ids=ids)
        if n:
            self.rebuild_needed = True
        return n

    # -- step, split in the two halves around the barrier (pipeline.py:905-940) --
    def step_pre_barrier(self, step):
        par = step & 1
        if self.options.rebuild == "every_step":
            self.rebuild_needed = True
        rebuilt = False
        if self.rebuild_needed:
            if self._pending_gather:
                self._flush_gather()
            self._rebuild(step, par)
            rebuilt = True
        else:
            self._clear(par)
        fused_now = self._fused_active()
        self.fused_mode = fused_now
        if fused_now and self._pending_gather:
            self._run_g2p2g(step, par)
        else:
            if self._pending_gather:
                self._flush_gather()
            self._run_p2g(step, par)
        codes, count = self._published_codes
        self.runtime.publish_step(par, self.wid, dict(
            raw=self.grid.raw[par], touched=self.table.touched[par], codes=codes,
            code_count=count, rebuilt=rebuilt))
        self._fused_now = fused_now

    def step_post_barrier(self, step):
        par = step & 1
        self._post_barrier(par)
        self._reduce_and_update(par)
        if self._fused_now:
            self._pending_gather = True
        else:
            self._run_g2p(step)
            self._pending_gather = False
        self.steps_since_rebuild += 1
        self._global_step = step + 1

    def run_step(self, step):
        assert self.runtime.n_workers == 1, "use OracleCluster for several workers"
        self.step_pre_barrier(step)
        self.runtime.generations += 1
        self.step_post_barrier(step)

    def run_frame(self):
        self._run_frame()
        if getattr(self, "_sunk_pending", False):
            self._sunk_pending = False
            self.rebuild_needed = True

    def _run_frame(self):
        """pipeline.py:856-880 (single worker)."""
        self.frame_steps = 0
        if self.cfl_mode:
            c_sound = sound_speed(self.material)
            t = 0.0
            while t < self.params.frame_dt - 1e-12:
                vmax = self.runtime.global_vmax((self._global_step - 2) % 3)
                self.dt = cfl_dt(vmax + c_sound, self.params, self.params.frame_dt - t)
                self.run_step(self._global_step)
                t += self.dt
                self.frame_steps += 1
        else:
            self.dt = self.params.dt
            for _ in range(self.params.steps_per_frame):
                self.run_step(self._global_step)
                self.frame_steps += 1
        if self._pending_gather:
            self._flush_gather()

    # -- phases --
    def _fused_active(self):
        if self.options.transfer != "g2p2g":
            return False
        if self.store.staged_count:
            return False
        if self.store.count >= self.options.fused_threshold:
            return False
        return True

    def _rebuild(self, step, par):
        st = self.store
        flat, ids = st.gather_flat()
        n = len(ids)
        codes = particle_code_batch(flat[:, CH_POS:CH_POS + 3], self.params.dx) if n \
            else np.empty(0, dtype=np.int64)
        gidx = self.table.rebuild(codes >> 6)
        keys = (gidx << 6) | (codes & 63)
        perm = st.histogram_sort(flat, ids, keys)
        self.last_perm, self.last_gidx = perm, gidx
        if st.n_groups:
            bcodes = self.table.codes[st.group_block[:st.n_groups].astype(np.int64)]
            st.group_origin[:st.n_groups] = (4 * decode_batch(bcodes)).astype(np.int32)
            st.refresh_lane_keys(self.params.dx)
        count = self.table.count
        g = self.grid
        g.vel = np.zeros((count, 4, 64))
        g.raw[par] = np.zeros((count, 4, 64))
        g.raw[1 - par] = _resize_rows(g.raw[1 - par], count)
        if g.vel_old is not None:
            g.vel_old = _resize_rows(g.vel_old, count)
        g.count = count
        self.table.touched[par][:count] = 0
        self._pending_full_clear_parity = 1 - par
        self._published_codes = (self.table.codes[:count].copy(), count)
        self.rebuild_needed = False
        self.steps_since_rebuild = 0
        self.rebuild_steps.append(step)

    def _clear(self, par):
        count = self.table.count
        raw = self.grid.raw[par]
        t = self.table.touched[par]
        if self._pending_full_clear_parity == par:
            raw[:count] = 0.0
            t[:count] = 0
            self._pending_full_clear_parity = -1
        else:
            idx = np.flatnonzero(t[:count])
            if len(idx):
                raw[idx] = 0.0
                t[idx] = 0

    def _run_p2g(self, step, par):
        st = self.store
        if not st.n_groups:
            return
        lib().orc_p2g(_p(st.data), _p(st.lane_key), _p(st.quarantined), _p(st.group_len),
                      _p(st.group_block), _p(st.group_origin), _i(st.n_groups),
                      _p(self.table.neighbor), _p(self.grid.raw[par]), _p(self.table.touched[par]),
                      C.byref(self._tp), _d(self.dt), _p(self.counters))
        self._check_addressing()

    def _vel_old_arg(self):
        save_old = self.params.flip_blend > 0.0
        g = self.grid
        if save_old and g.vel_old is None:
            g.vel_old = np.zeros((self.table.count, 3, 64))
        return g.vel_old if save_old else g.vel

    def _run_g2p(self, step):
        st = self.store
        vel_old = self._vel_old_arg()
        if not st.n_groups:
            self.runtime.publish_vmax(step % 3, self.wid, 0.0)
            return
        stats = np.zeros(3)
        lib().orc_gather_advect(
            _p(st.data), _p(st.lane_key), _p(st.quarantined), _p(st.group_len), _p(st.group_block),
            _p(st.group_origin), _p(self.table.neighbor), _p(self.grid.vel), _p(vel_old),
            _d(self.params.flip_blend), C.byref(self._tp), _d(self._vel_dt), _i(CELL_BIAS),
            _d(FREE_ZONE_LO_CELLS), _d(FREE_ZONE_HI_CELLS - 4.0), _i(0), _i(st.n_groups),
            _p(stats), _p(self.counters))
        self._check_addressing()
        if stats[0] > 0.0:
            self.rebuild_needed = True
        self._after_gather_stats(stats)
        self.runtime.publish_vmax(step % 3, self.wid, float(np.sqrt(stats[1])))

    def _flush_gather(self):
        self._run_g2p(self._global_step)
        self._pending_gather = False

    def _run_g2p2g(self, step, par):
        st = self.store
        vel_old = self._vel_old_arg()
        if not st.n_groups:
            return
        stats = np.zeros(3)
        lib().orc_g2p2g(
            _p(st.data), _p(st.lane_key), _p(st.quarantined), _p(st.group_len), _p(st.group_block),
            _p(st.group_origin), _i(st.n_groups), _p(self.table.neighbor), _p(self.grid.vel),
            _p(vel_old), _d(self.params.flip_blend), _p(self.grid.raw[par]),
            _p(self.table.touched[par]), C.byref(self._tp), _d(self._vel_dt), _d(self.dt),
            _i(CELL_BIAS), _d(FREE_ZONE_LO_CELLS - FUSED_MARGIN_CELLS),
            _d(FREE_ZONE_HI_CELLS - 4.0 - FUSED_MARGIN_CELLS), _p(stats), _p(self.counters))
        self._check_addressing()
        if stats[0] > 0.0:
            self.rebuild_needed = True
        self._after_gather_stats(stats)
        self.runtime.publish_vmax(step % 3, self.wid, float(np.sqrt(stats[1])))

    def _post_barrier(self, par):
        if self.runtime.n_workers == 1:
            return
        states = [self.runtime.peer_step(par, q) for q in range(self.runtime.n_workers)]
        if any(s["rebuilt"] for s in states):
            for q, s in enumerate(states):
                if q == self.wid:
                    continue
                idx = self.table.hash.lookup_batch(s["codes"][:s["code_count"]])
                m = np.full(self.table.count, -1, dtype=np.int64)
                found = np.flatnonzero(idx >= 0)
                m[idx[found]] = found
                self._peer_map[q] = m
        self._peer_states = states

    def _reduce_and_update(self, par):
        count = self.table.count
        touched_idx = np.ascontiguousarray(np.flatnonzero(self.table.touched[par][:count]),
                                           dtype=np.int64)
        vel, raw = self.grid.vel, self.grid.raw[par]
        L = lib()
        L.orc_copy_rows(_p(vel), _p(raw), _p(touched_idx), _i(len(touched_idx)))
        if self.runtime.n_workers > 1 and self._peer_states is not None and len(touched_idx):
            for q, s in enumerate(self._peer_states):
                if q == self.wid or self._peer_map[q] is None:
                    continue
                L.orc_add_peer_rows(_p(vel), _p(touched_idx), _i(len(touched_idx)),
                                    _p(self._peer_map[q]), _p(s["raw"]), _p(s["touched"]))
        if self.options.collect_conservation:
            det = self.options.deterministic
            if len(touched_idx):
                own = raw[touched_idx]
                gm = float(own[:, 0, :].sum())
                gmom = own[:, 1:4, :].sum(axis=(0, 2))
            else:
                gm, gmom = 0.0, np.zeros(3)
            if det:
                gm /= MASS_SCALE
                gmom = gmom / MOM_SCALE
            self.conservation.append((self.store.total_mass(), *self.store.total_momentum(),
                                      gm, *gmom))
        grav = np.array(self.params.gravity, dtype=np.float64)
        bc = self.boundary
        save_old = self.params.flip_blend > 0.0
        if save_old:
            self.grid.vel_old = np.zeros((count, 3, 64)) if self.grid.vel_old is None \
                else _resize_rows(self.grid.vel_old, count)
        vel_old = self.grid.vel_old if save_old else vel
        if bc is not None:
            blo = np.array(bc.min_corner, dtype=np.float64)
            bhi = np.array(bc.max_corner, dtype=np.float64)
            sticky = bc.mode == "sticky"
        else:
            blo, bhi, sticky = np.full(3, -1e30), np.full(3, 1e30), False
        L.orc_grid_finalize(_p(vel), _p(touched_idx), _i(len(touched_idx)), _p(self.table.codes),
                            _i(self.options.deterministic), _d(self.dt), _p(grav), _p(blo),
                            _p(bhi), _i(sticky), _i(bc is not None), _d(self.params.dx),
                            _i(CELL_BIAS), _p(vel_old), _i(save_old))
        self._vel_dt = self.dt

    def _check_addressing(self):
        if self.counters[C_ADDRESS_ERR]:
            raise OracleContractViolation(
                f"worker {self.wid}: {int(self.counters[C_ADDRESS_ERR])} stencil accesses left "
                f"the 27-neighbor pblock set")


class OracleCluster:
    """n workers stepped in lockstep; optional thread pool so the per-phase C calls of
    different workers run on different cores (ctypes releases the GIL)."""

    def __init__(self, n, params, material, boundary, options=None, initial_vmax=0.0,
                 threads=False):
        self.runtime = OracleRuntime(n, initial_vmax)
        # one Material per worker = material populations sharing the grid (not in the reference,
        # which has one material per run; the grid reduction is pipeline.py:1172-1188 unchanged)
        materials = list(material) if isinstance(material, (list, tuple)) else [material] * n
        self.workers = [OracleWorker(w, self.runtime, params, materials[w], boundary, options)
                        for w in range(n)]
        self.params = params
        self.threads = threads and n > 1
        self.cfl_mode = False
        self.frame_steps = 0

    def seed(self, positions, velocities, mass):
        parts = partition_particles(positions, len(self.workers))
        for w, part in zip(self.workers, parts):
            if len(part):
                w.seed_particles(positions[part], velocities[part], mass, ids=part)
        return parts

    def seed_populations(self, populations):
        base = 0
        for w, pop in zip(self.workers, populations):
            n = len(pop[0])
            ids = np.asarray(pop[3], dtype=np.int64) if len(pop) > 3 else np.arange(base, base + n, dtype=np.int64)
            if n:
                w.seed_particles(pop[0], pop[1], pop[2], ids=ids)
            base += n

    def _phase(self, fn):
        if not self.threads:
            for w in self.workers:
                fn(w)
            return
        errs = []

        def run(w):
            try:
                fn(w)
            except BaseException as e:  # noqa
                errs.append(e)
        ts = [threading.Thread(target=run, args=(w,)) for w in self.workers]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]

    def run_step(self, step):
        self._phase(lambda w: w.step_pre_barrier(step))
        self.runtime.generations += 1
        self._phase(lambda w: w.step_post_barrier(step))

    def run_frame(self):
        ws = self.workers
        self.frame_steps = 0
        if self.cfl_mode:
            c_sound = max(sound_speed(w.material) for w in ws)
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

    def positions_sorted_by_id(self):
        chunks = [w.store.positions_with_ids() for w in self.workers]
        pos = np.concatenate([c[0] for c in chunks], axis=0)
        ids = np.concatenate([c[1] for c in chunks], axis=0)
        return pos[np.argsort(ids, kind="stable")]

    def state_sorted_by_id(self):
        chunks = [w.store.state_with_ids() for w in self.workers]
        nch = max(c[0].shape[1] for c in chunks)
        chunks = [(np.pad(c[0], ((0, 0), (0, nch - c[0].shape[1]))), c[1]) for c in chunks]
        flat = np.concatenate([c[0] for c in chunks], axis=0)
        ids = np.concatenate([c[1] for c in chunks], axis=0)
        return flat[np.argsort(ids, kind="stable")]
