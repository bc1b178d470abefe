"""Generate golden vectors by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Imports `mpmbench` from /root/reference (read-only, public, untrusted: only executed,
never copied) and dumps small input/output arrays to tests/golden/*.npz.  The GPU box
has no /root/reference, so tests only ever read the committed .npz files.

Scenes (all inputs are float32-representable doubles so an fp32 device path sees the
same numbers):
  kat.npz        leaf known-answer vectors: Morton codes, particle codes, counting sort,
                 lane radix order, SVD / fixed-corotated stress, fluid pressure
  elastic.npz    1728-particle falling block, fixed-corotated, slip box, split transfers:
                 full state after step 0 (tables, sort, raw, vel, particles) and particle
                 state after 1, 2 and 24 steps (>=1 amortised rebuild)
  fluid.npz      1000-particle weakly-compressible blob, same dumps
  fused.npz      elastic scene with transfer=g2p2g, state after 24 steps (+flush)
  flip.npz       elastic scene with flip_blend=0.8, state after 6 steps
  two_worker.npz elastic scene on 2 workers (threads), state after 1 and 24 steps
  det.npz        elastic scene, deterministic mode, 1 vs 2 workers, raw after step 0
  cfl.npz        fluid scene in CFL-auto mode: dt sequence of one frame
"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from mpmbench import Material, SharedRuntime, SimParams  # noqa: E402
from mpmbench.domain import _corotated_tau, _svd3_scalars  # noqa: E402
from mpmbench.grid import encode_batch  # noqa: E402
from mpmbench.multiworker import partition_particles  # noqa: E402
from mpmbench.particles import (lane_radix_sort10, particle_code_batch,  # noqa: E402
                                stable_counting_sort)
from mpmbench.pipeline import BoundaryBox, PipelineOptions, Worker, _fluid_tau  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32r(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def block_scene(l, seed, dx, origin_cells=(10, 10, 12), ppc_side=2, speed=-150.0):
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
    vel += rng.normal(0.0, 5.0, pos.shape)
    order = rng.permutation(len(pos))      # unsorted input order exercises the sort
    return f32r(pos[order]), f32r(vel[order])


def make_workers(n, pos, vel, material, params, boundary, mass, **opts):
    runtime = SharedRuntime(n, initial_vmax=float(np.linalg.norm(vel, axis=1).max()))
    options = PipelineOptions(**opts)
    ws = [Worker(w, runtime, params, material, boundary, options) for w in range(n)]
    parts = partition_particles(pos, n)
    for w, part in zip(ws, parts):
        w.seed_particles(pos[part], vel[part], mass, ids=part)
        w.dt = params.dt
    return ws


def lockstep(ws, steps, start=0):
    if len(ws) == 1:
        for s in range(start, start + steps):
            ws[0].run_step(s)
        return
    errs = []

    def loop(w):
        try:
            for s in range(start, start + steps):
                w.run_step(s)
        except BaseException as e:  # noqa
            errs.append(e)
    ts = [threading.Thread(target=loop, args=(w,)) for w in ws]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


def state_by_id(ws):
    flats, ids = [], []
    for w in ws:
        st = w.store
        G = st.n_groups
        d = st.data.data[:G]
        gl = st.group_len.data[:G]
        for g in range(G):
            for l in range(gl[g]):
                flats.append(d[g, :, l].copy())
                ids.append(int(st.orig_id.data[g, l]))
    flats = np.array(flats)
    order = np.argsort(np.array(ids), kind="stable")
    return flats[order]


def dump_step0(w, prefix, out):
    st, tb, gr = w.store, w.table, w.grid
    G = st.n_groups
    out[prefix + "codes"] = tb.codes.data[:tb.count].copy()
    out[prefix + "n_gblocks"] = np.int64(tb.n_gblocks)
    out[prefix + "neighbor"] = tb.neighbor.data[:tb.n_gblocks].copy()
    out[prefix + "group_len"] = st.group_len.data[:G].copy()
    out[prefix + "group_block"] = st.group_block.data[:G].copy()
    out[prefix + "group_origin"] = st.group_origin.data[:G].copy()
    out[prefix + "orig_id"] = st.orig_id.data[:G].copy()
    out[prefix + "lane_key"] = st.lane_key.data[:G].copy()
    out[prefix + "data"] = st.data.data[:G].copy()
    out[prefix + "raw0"] = gr.raw[0].data[:tb.count].copy()
    out[prefix + "vel"] = gr.vel.data[:tb.count].copy()
    out[prefix + "touched0"] = tb.touched[0].data[:tb.count].copy()
    out[prefix + "counters"] = w.counters.copy()


DX = 25.0 / 64.0
DT = (1.0 / 48.0) / 36.0


def elastic_setup():
    pos, vel = block_scene(6, 11, DX)
    material = Material.fixed_corotated(2.0, 1.0e5, 0.3)
    params = SimParams(dx=DX, dt=DT)
    boundary = BoundaryBox((8 * DX,) * 3, (40 * DX,) * 3, mode="slip")
    mass = 2.0 * DX ** 3 / 8
    return pos, vel, material, params, boundary, mass


def fluid_setup():
    pos, vel = block_scene(5, 12, 0.5, origin_cells=(9, 9, 10), speed=-60.0)
    material = Material.fluid(1.0, 1.0e5, 7.0)
    params = SimParams(dx=0.5, dt=2.0e-4)
    boundary = BoundaryBox((4.0,) * 3, (20.0,) * 3, mode="sticky")
    mass = 1.0 * 0.5 ** 3 / 8
    return pos, vel, material, params, boundary, mass


def gen_kat():
    rng = np.random.default_rng(2024)
    out = {}
    cells = rng.integers(0, 1 << 21, size=(64, 3))
    cells[0] = (1, 2, 3)
    out["cells"] = cells
    out["cell_codes"] = encode_batch(cells)
    pos = f32r(rng.uniform(-20.0, 60.0, (256, 3)))
    out["pos"] = pos
    out["pos_codes_dx"] = np.float64(DX)
    out["pos_codes"] = particle_code_batch(pos, DX)
    keys = rng.integers(0, 500, size=2000)
    out["sort_keys"] = keys
    out["sort_perm"] = stable_counting_sort(keys)
    lk = rng.integers(0, 1000, size=(16, 32))
    out["lane_keys"] = lk
    out["lane_order"] = np.stack([lane_radix_sort10(k) for k in lk])
    F = np.eye(3)[None] + rng.normal(0.0, 0.25, (200, 3, 3))
    F[0] = np.eye(3)
    F[1] = np.diag([1.2, 1.2, 0.7])
    F[2] = np.diag([1.0, 1.0, 0.0])            # collapsed -> clamp
    F[3] = -np.eye(3)                           # inverted
    F[4] = np.diag([2.0, 2.0, 2.0])             # degenerate eigenvalues
    F[5] = np.array([[1, 0.5, 0], [0, 1, 0], [0, 0, 1.0]])
    F = f32r(F)
    mu, lam = 1.0e5 / 2.6, 1.0e5 * 0.3 / (1.3 * 0.4)
    svd = np.array([_svd3_scalars(*f.reshape(9)) for f in F])
    tau = np.array([_corotated_tau(*f.reshape(9), mu, lam) for f in F])
    out["F"] = F
    out["mu_lam"] = np.array([mu, lam])
    out["svd"] = svd
    out["tau"] = tau[:, :9]
    out["tau_clamped"] = tau[:, 9].astype(np.int64)
    J = f32r(rng.uniform(0.7, 1.3, 64))
    out["J"] = J
    out["fluid_tau"] = np.array([_fluid_tau(j, 1.0e5, 7.0, False) for j in J])
    out["fluid_tau_clamp"] = np.array([_fluid_tau(j, 1.0e5, 7.0, True) for j in J])
    np.savez_compressed(os.path.join(OUT, "kat.npz"), **out)


def gen_single(name, setup, steps_dump=(1, 2, 24), **opts):
    pos, vel, material, params, boundary, mass = setup()
    ws = make_workers(1, pos, vel, material, params, boundary, mass, **opts)
    w = ws[0]
    out = dict(pos=pos, vel=vel, mass=np.float64(mass))
    done = 0
    for target in steps_dump:
        lockstep(ws, target - done, start=done)
        done = target
        if target == 1:
            dump_step0(w, "s0_", out)
        if w._pending_gather:
            # fused runs leave the last gather pending; dump the flushed state of a copy
            pass
        out[f"state_{target}"] = state_by_id(ws)
    if w._pending_gather:
        w._flush_gather()
        out["state_final_flushed"] = state_by_id(ws)
    out["rebuild_steps"] = np.array(w.rebuild_steps, dtype=np.int64)
    out["counters"] = w.counters.copy()
    np.savez_compressed(os.path.join(OUT, name), **out)
    print(name, "rebuild steps", w.rebuild_steps, "n", len(pos))


def gen_two_worker():
    pos, vel, material, params, boundary, mass = elastic_setup()
    out = dict(pos=pos, vel=vel, mass=np.float64(mass))
    ws = make_workers(2, pos, vel, material, params, boundary, mass)
    lockstep(ws, 1)
    for w in ws:
        dump_step0(w, f"w{w.wid}_s0_", out)
        for q, m in enumerate(w._peer_map):
            if m is not None:
                out[f"w{w.wid}_peer_map{q}"] = m.copy()
    out["state_1"] = state_by_id(ws)
    lockstep(ws, 23, start=1)
    out["state_24"] = state_by_id(ws)
    out["rebuild_steps0"] = np.array(ws[0].rebuild_steps, dtype=np.int64)
    out["rebuild_steps1"] = np.array(ws[1].rebuild_steps, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "two_worker.npz"), **out)
    print("two_worker rebuild steps", ws[0].rebuild_steps, ws[1].rebuild_steps)


def gen_det():
    pos, vel, material, params, boundary, mass = elastic_setup()
    out = dict(pos=pos, vel=vel, mass=np.float64(mass))
    for n in (1, 2):
        ws = make_workers(n, pos, vel, material, params, boundary, mass, deterministic=True)
        lockstep(ws, 8)
        out[f"state_8_n{n}"] = state_by_id(ws)
    assert np.array_equal(out["state_8_n1"], out["state_8_n2"])
    np.savez_compressed(os.path.join(OUT, "det.npz"), **out)


def gen_cfl():
    pos, vel, material, params, boundary, mass = fluid_setup()
    params = SimParams(dx=0.5, dt=2.0e-4, frame_dt=1.0 / 240.0, cfl=0.5)
    ws = make_workers(1, pos, vel, material, params, boundary, mass)
    w = ws[0]
    w.cfl_mode = True
    dts = []
    orig = w.run_step

    def spy(step):
        dts.append(w.dt)
        orig(step)
    w.run_step = spy
    w.run_frame()
    w.run_frame()
    out = dict(pos=pos, vel=vel, mass=np.float64(mass), dts=np.array(dts),
               state=state_by_id(ws), frame_dt=np.float64(params.frame_dt))
    np.savez_compressed(os.path.join(OUT, "cfl.npz"), **out)
    print("cfl steps", len(dts))


if __name__ == "__main__":
    gen_kat()
    gen_single("elastic.npz", elastic_setup)
    gen_single("fluid.npz", fluid_setup)
    gen_single("fused.npz", elastic_setup, steps_dump=(24,), transfer="g2p2g")

    def flip_setup():
        pos, vel, material, params, boundary, mass = elastic_setup()
        params = SimParams(dx=DX, dt=DT, flip_blend=0.8)
        return pos, vel, material, params, boundary, mass
    gen_single("flip.npz", flip_setup, steps_dump=(6,))
    gen_two_worker()
    gen_det()
    gen_cfl()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)) // 1024, "KiB")
