"""ctypes binding of libmpm_b200.so (include/mpm_b200.h).

The library is the product path: if it is missing, or the CUDA device is not a B200-class
part when a compute call is made, this module raises -- there is no CPU fallback.
Status codes map 1:1 onto the reference's exception classes
(/root/reference/pkg/src/mpmbench/errors.py:4-37).
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPM_B200_LIB", os.path.join(_HERE, "libmpm_b200.so"))   # override: kernel experiments

MPM_MAX_PEERS = 15
N_COUNTERS = 6
LANE_QUARANTINED = 0x8000
LANE_SUNK = 0x4000

p_void = C.c_void_p
i32 = C.c_int32
f64 = C.c_double


class TransferParams(C.Structure):
    _fields_ = [
        ("mat_kind", i32), ("nch", i32),
        ("mu", f64), ("lam", f64), ("kappa", f64), ("gamma", f64),
        ("clamp_tension", i32), ("count_stats", i32), ("deterministic", i32), ("reserved0", i32),
        ("density", f64), ("dx", f64), ("dt", f64), ("dt_gather", f64), ("flip_blend", f64),
        ("margin_lo", f64), ("margin_hi", f64),
        ("theta_c", f64), ("theta_s", f64), ("hardening", f64), ("sand_alpha", f64),
        ("clock", p_void), ("clock_step", i32), ("clock_gather_step", i32),
        ("sink_enabled", i32), ("reserved5", i32), ("sink_lo", f64 * 3), ("sink_hi", f64 * 3),
    ]


class StoreView(C.Structure):
    _fields_ = [
        ("data", p_void), ("orig_id", p_void), ("lane_meta", p_void), ("group_len", p_void),
        ("group_block", p_void), ("group_start", p_void), ("n_groups", i32), ("nch", i32),
        ("group_ctx", p_void), ("n_groups_dev", p_void),
    ]


class TableView(C.Structure):
    _fields_ = [
        ("codes", p_void), ("origin", p_void), ("neighbor", p_void), ("touched", p_void * 2),
        ("count", i32), ("n_gblocks", i32), ("count_dev", p_void),
    ]


class GridParams(C.Structure):
    _fields_ = [
        ("dt", f64), ("gravity", f64 * 3), ("apply_bc", i32), ("bc_sticky", i32),
        ("box_lo", f64 * 3), ("box_hi", f64 * 3), ("dx", f64), ("fuse_clear", i32),
        ("block_filter", i32), ("deterministic", i32), ("n_peers", i32),
        ("peer_raw", p_void * MPM_MAX_PEERS), ("peer_touched", p_void * MPM_MAX_PEERS),
        ("peer_map", p_void * MPM_MAX_PEERS),
        ("n_wait", i32), ("wait_value", i32), ("wait_timeout_ms", i32), ("reserved1", i32),
        ("wait_flags", p_void * MPM_MAX_PEERS), ("wait_error", p_void),
        ("publish_src", p_void), ("publish_dst", p_void), ("publish_guard_src", p_void),
        ("publish_guard_dst", p_void),
        ("clock", p_void), ("clock_step", i32), ("vmax_ring_len", i32), ("vmax_ring", p_void),
        ("clock_status", p_void), ("frame_dt", f64), ("cfl_dx", f64), ("c_sound", f64),
        ("n_vmax_peers", i32), ("reserved4", i32), ("vmax_peer_rings", p_void * MPM_MAX_PEERS),
        ("prof", p_void),
    ]


class Guard(C.Structure):
    _fields_ = [("first_bad_step", p_void), ("step", i32), ("n_peer_words", i32),
                ("peer_words", p_void * MPM_MAX_PEERS)]


class StepStatus(C.Structure):
    _fields_ = [("zone_violation", i32), ("vmax2_bits", C.c_uint32),
                ("counters", C.c_ulonglong * N_COUNTERS), ("dt", f64), ("removed", C.c_ulonglong)]


class StepClock(C.Structure):
    _fields_ = [("dt", f64 * 2), ("t", f64), ("reserved", f64)]


STATUS_ZONE, STATUS_FRAME_END = 1, 2


STATUS_BYTES = C.sizeof(StepStatus)
MAX_STATUS_RING = 32


class StepPlan(C.Structure):
    _fields_ = [
        ("store", StoreView), ("table", TableView), ("raw", p_void * 2), ("touched", p_void * 2),
        ("vel", p_void), ("vel_old", p_void), ("transfer", TransferParams),
        ("fused_margin_lo", f64), ("fused_margin_hi", f64), ("grid", GridParams),
        ("fused", i32), ("status_ring", i32), ("status_dev", p_void), ("status_host", p_void),
        ("events", p_void * MAX_STATUS_RING), ("guard_word", p_void),
        ("n_peer_words", i32), ("reserved2", i32), ("peer_guard_words", p_void * MPM_MAX_PEERS),
        ("signal_word", p_void), ("guard_host", p_void),
        ("peer_raw", (p_void * MPM_MAX_PEERS) * 2), ("peer_touched", (p_void * MPM_MAX_PEERS) * 2),
        ("time_events", p_void * (2 * MAX_STATUS_RING)),
        ("full_clear_first", i32), ("reserved3", i32),
    ]


class RebuildPlan(C.Structure):
    _fields_ = [
        ("old_store", StoreView), ("new_store", StoreView), ("cap_groups", i32), ("n_staged", i32),
        ("staged", p_void), ("staged_ids", p_void), ("n_upper", i32), ("cap_gblocks", i32), ("dx", f64),
        ("glive", p_void), ("src_slot", p_void), ("pslot", p_void), ("flag", p_void), ("gidx", p_void),
        ("tmp_perm", p_void), ("perm", p_void), ("codes", p_void), ("gcodes", p_void), ("scan", p_void),
        ("qslot", p_void), ("qflag", p_void), ("bin_start", p_void), ("bgf", p_void),
        ("hkeys", p_void), ("hvals", p_void), ("hfirst", p_void), ("hash_cap", i32), ("cap_table", i32),
        ("table_codes", p_void), ("table_origin", p_void), ("table_neighbor", p_void),
        ("vel", p_void), ("raw_par", p_void), ("touched_par", p_void), ("cap_nodes", i32),
        ("node_bytes", i32), ("scalars_dev", p_void), ("scalars_host", p_void),
        ("p2g_params", p_void), ("p2g_status", p_void), ("grid_params", p_void),
        ("grid_reset_status", p_void), ("vel_old", p_void), ("guard_word", p_void),
        ("guard_step", i32), ("async_", i32), ("large_list", p_void), ("done_event", p_void),
        ("g2p_params", p_void), ("g2p_status", p_void), ("status_publish_dst", p_void),
        ("status_event", p_void), ("next_steps", p_void), ("next_first_step", i32), ("next_n_steps", i32),
        ("n_groups_out", p_void), ("use_graph", i32), ("reserved1", i32),
    ]


class RebuildResult(C.Structure):
    _fields_ = [(k, i32) for k in ("n", "n_gblocks", "count", "n_groups", "bad_particle", "bad_block",
                                   "need_hash", "need_gblocks", "need_table", "need_groups",
                                   "need_nodes", "tail_done", "g2p_done", "next_done", "graph")]


NEED_CAPACITY = 1
SHM_MAX_VALUES = 15

_STATUS_TO_ERROR = {
    -1: E.RejectedInputError, -2: E.SpatialDomainError, -3: E.ResourceError,
    -4: E.ContractViolationError, -5: E.ModeConflictError, -6: E.DegenerateStateError,
    -7: E.ConfigError, -8: E.BarrierTimeoutError,
}

# name -> argtypes; every function returns int (mpm_status) unless listed in _RESTYPES
_SIGNATURES = {
    "mpm_fill_i32": [p_void, i32, i32, p_void],
    "mpm_stage_particles": [p_void, p_void, p_void, C.c_float, i32, i32, i32, p_void, p_void],
    "mpm_compact_live": [C.POINTER(StoreView), i32, p_void, p_void, p_void, p_void, p_void],
    "mpm_particle_codes": [C.POINTER(StoreView), p_void, p_void, p_void, i32, i32, f64, p_void,
                           p_void, p_void, p_void],
    "mpm_hash_insert_blocks": [p_void, p_void, i32, p_void, p_void, p_void, i32, p_void, p_void,
                               p_void, p_void, p_void, p_void, p_void, p_void],
    "mpm_dilate_and_link": [p_void, p_void, i32, p_void, p_void, p_void, i32, p_void, p_void, p_void,
                            p_void, p_void, p_void, i32, p_void, p_void, p_void, p_void],
    "mpm_sort_and_group": [p_void, p_void, p_void, i32, p_void, i32, p_void, p_void, p_void, p_void,
                           p_void, p_void, p_void, p_void, p_void],
    "mpm_scatter_sorted": [C.POINTER(StoreView), p_void, p_void, p_void, p_void, p_void, p_void,
                           p_void, p_void, p_void, f64, C.POINTER(StoreView), p_void, p_void],
    "mpm_build_group_ctx": [C.POINTER(StoreView), C.POINTER(TableView), p_void],
    "mpm_rebuild": [C.POINTER(RebuildPlan), C.POINTER(RebuildResult), p_void],
    "mpm_rebuild_wait": [C.POINTER(RebuildPlan), C.POINTER(RebuildResult)],
    "mpm_clear": [p_void, p_void, i32, i32, i32, C.POINTER(Guard), p_void],
    "mpm_status_reset": [p_void, C.POINTER(Guard), p_void],
    "mpm_status_publish": [p_void, p_void, p_void, p_void, p_void],
    "mpm_p2g": [C.POINTER(StoreView), C.POINTER(TableView), p_void, p_void,
                C.POINTER(TransferParams), p_void, C.POINTER(Guard), p_void],
    "mpm_grid_update": [p_void, p_void, p_void, p_void, C.POINTER(TableView),
                        C.POINTER(GridParams), p_void, C.POINTER(Guard), p_void],
    "mpm_pack_halo": [p_void, p_void, p_void, i32, p_void, p_void],
    "mpm_signal_step": [p_void, i32, C.POINTER(Guard), p_void],
    "mpm_wait_step": [C.POINTER(GridParams), C.POINTER(Guard), p_void],
    "mpm_g2p": [C.POINTER(StoreView), C.POINTER(TableView), p_void, p_void,
                C.POINTER(TransferParams), p_void, C.POINTER(Guard), p_void],
    "mpm_g2p2g": [C.POINTER(StoreView), C.POINTER(TableView), p_void, p_void, p_void, p_void,
                  C.POINTER(TransferParams), p_void, C.POINTER(Guard), p_void],
    "mpm_enqueue_steps": [C.POINTER(StepPlan), i32, i32, p_void],
    "mpm_gather_state": [C.POINTER(StoreView), p_void, p_void, p_void],
    "mpm_gather_positions": [C.POINTER(StoreView), p_void, p_void, p_void],
    "mpm_particle_aggregates": [C.POINTER(StoreView), p_void, p_void],
    "mpm_grid_aggregates": [p_void, p_void, i32, i32, p_void, p_void],
    "mpm_tag_shared": [p_void, i32, p_void, p_void, i32, p_void, i32, p_void],
    "mpm_version": [],
    "mpm_last_error": [],
    "mpm_device_arch": [],
    "mpm_launch_count": [],
    "mpm_host_alias": [p_void],
    "mpm_ipc_open": [C.c_char_p, C.POINTER(p_void)],
    "mpm_ipc_close": [p_void],
    "mpm_peek_i32": [p_void, p_void],
    "mpm_shm_bytes": [i32],
    "mpm_shm_allgather_i64": [p_void, i32, i32, p_void, i32, p_void, i32],
}
_RESTYPES = {"mpm_version": C.c_char_p, "mpm_last_error": C.c_char_p,
             "mpm_launch_count": C.c_ulonglong, "mpm_host_alias": C.c_void_p, "mpm_shm_bytes": C.c_int64}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def lib() -> C.CDLL:
    """Load libmpm_b200.so (built by paper_2111_00699_b200.build).  Raises ResourceError when
    the library is missing: the CUDA core is the only implementation of the substep."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise E.ResourceError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2111_00699_b200.build` "
                "(there is no CPU fallback for the substep)")
        handle = C.CDLL(LIB_PATH)
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = handle
    return _lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    cls = _STATUS_TO_ERROR.get(status, E.SimulationError)
    detail = lib().mpm_last_error().decode() if status == -3 else ""
    raise cls(f"{what or 'libmpm_b200'} failed with status {status} {detail}".strip())


def require_device() -> None:
    """Fail loudly unless a CUDA device of compute capability 10.x is current."""
    import torch
    if not torch.cuda.is_available():
        raise E.ResourceError("no CUDA device: the MLS-MPM substep core is CUDA-only (sm_100a)")
    arch = lib().mpm_device_arch()
    if arch // 10 != 10:
        raise E.ResourceError(f"libmpm_b200.so is built for sm_100a; current device is sm_{arch}")
