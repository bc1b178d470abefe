"""Helpers shared by the GPU parity tests: build the CUDA worker and the oracle on the same
inputs, and measure the differences per quantity with the tolerances written down here.

Tolerances (fp32 device path vs the float64 reference/oracle), per north_star:
  * block assignment / sort permutation / lane structure: BIT-EXACT
  * grid mass & momentum after one substep: max-abs error <= GRID_RTOL * max|channel|
  * particle x / v / F after one substep: X_RTOL * domain edge, V_RTOL * max|v|, F_ATOL
  * after a short run the same quantities with the *_RUN tolerances (error accumulates
    through F <- (I + dt C) F and advection), and aggregate drift (total mass, momentum,
    kinetic energy) <= AGG_RTOL.
"""
import numpy as np

from oracle import mpm_oracle as O
from paper_2111_00699_b200 import PipelineOptions

GRID_RTOL = 1e-5
X_RTOL = 1e-6
V_RTOL = 1e-5
F_ATOL = 1e-5
X_RTOL_RUN = 2e-5
V_RTOL_RUN = 2e-3
F_ATOL_RUN = 2e-3
AGG_RTOL = 1e-4

CH_POS, CH_VEL, CH_C, CH_MASS, CH_DEF = 0, 3, 6, 15, 16


def oracle_worker(pos, vel, mass, material, params, boundary, **opts):
    rt = O.OracleRuntime(1, float(np.linalg.norm(vel, axis=1).max()) if len(vel) else 0.0)
    w = O.OracleWorker(0, rt, params, material, boundary, PipelineOptions(**opts))
    part = O.partition_particles(pos, 1)[0] if len(pos) else np.zeros(0, dtype=np.int64)
    if len(pos):
        w.seed_particles(pos[part], vel[part], mass, ids=part)
    return w


def cuda_worker(pos, vel, mass, material, params, boundary, worker_kw=None, **opts):
    from paper_2111_00699_b200 import SharedRuntime
    from paper_2111_00699_b200.worker import CudaWorker
    rt = SharedRuntime(1, initial_vmax=float(np.linalg.norm(vel, axis=1).max()) if len(vel) else 0.0)
    w = CudaWorker(0, rt, params, material, boundary, PipelineOptions(**opts), **(worker_kw or {}))
    part = O.partition_particles(pos, 1)[0] if len(pos) else np.zeros(0, dtype=np.int64)
    if len(pos):
        w.seed_particles(pos[part], vel[part], mass, ids=part)
    return w


def state_by_id(w):
    flat, ids = w.store.state_with_ids()
    return flat[np.argsort(ids, kind="stable")]


def rel_err(got, ref):
    """max |got - ref| / max |ref| (0 when both are all-zero)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = np.abs(ref).max() if ref.size else 0.0
    err = np.abs(got - ref).max() if ref.size else 0.0
    return err / scale if scale > 0 else err


def grid_errors(got, ref):
    """per-channel relative errors of a [count, 4, 64] nodal buffer."""
    return [rel_err(got[:, c, :], ref[:, c, :]) for c in range(4)]


def particle_errors(got, ref, edge, nch_def):
    """(x error / edge, v error / max|v|, max abs F|J error, max abs C error / max|C|)."""
    ex = np.abs(got[:, CH_POS:CH_POS + 3] - ref[:, CH_POS:CH_POS + 3]).max() / edge
    ev = rel_err(got[:, CH_VEL:CH_VEL + 3], ref[:, CH_VEL:CH_VEL + 3])
    ef = np.abs(got[:, CH_DEF:CH_DEF + nch_def] - ref[:, CH_DEF:CH_DEF + nch_def]).max()
    ec = rel_err(got[:, CH_C:CH_C + 9], ref[:, CH_C:CH_C + 9])
    return ex, ev, ef, ec


def structure_mismatches(w, g, prefix="s0_"):
    """Names of the bit-exact structures that differ from a golden step-0 dump."""
    st, tb = w.store, w.table
    bad = []

    def eq(name, got):
        ref = g[prefix + name]
        if got.shape != ref.shape or not np.array_equal(got, ref):
            bad.append(name)
    eq("codes", tb.codes)
    if tb.n_gblocks != int(g[prefix + "n_gblocks"]):
        bad.append("n_gblocks")
    eq("neighbor", tb.neighbor)
    eq("group_len", st.group_len)
    eq("group_block", st.group_block)
    eq("group_origin", st.group_origin)
    eq("orig_id", st.orig_id)
    eq("lane_key", st.lane_key)
    eq("touched0", tb.touched[0])
    return bad


def block_scene(l, seed, dx, origin_cells=(10, 10, 12), ppc_side=2, speed=-150.0, jitter=5.0):
    """Same generator as tests/golden/make_golden.py::block_scene (float32-representable)."""
    rng = np.random.default_rng(seed)
    s = ppc_side
    cells = np.stack(np.meshgrid(np.arange(l), np.arange(l), np.arange(l), indexing="ij"),
                     axis=-1).reshape(-1, 3)
    subs = np.stack(np.meshgrid(np.arange(s), np.arange(s), np.arange(s), indexing="ij"),
                    axis=-1).reshape(-1, 3)
    base = (cells[:, None, :] * s + subs[None, :, :]).reshape(-1, 3)
    u = rng.random((base.shape[0], 3))
    pos = (np.asarray(origin_cells) + (base + u) / s) * dx
    vel = np.zeros_like(pos)
    vel[:, 2] = speed
    vel += rng.normal(0.0, jitter, pos.shape)
    order = rng.permutation(len(pos))
    f32r = lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)
    return f32r(pos[order]), f32r(vel[order])
