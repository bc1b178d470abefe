"""The reference's pipeline known-answer tests (pkg/tests/test_pipeline.py) restated on the
CUDA worker; each test cites the reference test it follows.  Values that are exact in float64
are checked at fp32 resolution here."""
import numpy as np
import pytest

from oracle import mpm_oracle as O
from paper_2111_00699_b200 import (BoundaryBox, Material, ModeConflictError, PipelineOptions,
                                   SimParams, SpatialDomainError)

pytestmark = pytest.mark.gpu

CH_VEL, CH_C, CH_MASS = 3, 6, 15
CELL_BIAS = 64


def _mk(pos, vel=None, *, material=None, params=None, boundary=None, mass=1.0, **opts):
    from paper_2111_00699_b200 import make_single_worker
    pos = np.atleast_2d(np.asarray(pos, dtype=np.float64)).reshape(-1, 3)
    vel = np.zeros_like(pos) if vel is None else np.atleast_2d(np.asarray(vel, dtype=np.float64))
    material = material or Material.fixed_corotated(2.0, 1.0e5, 0.3)
    params = params or SimParams(dx=0.5, dt=1e-4)
    return make_single_worker(pos, vel, material, params, boundary, mass, **opts)


def node_positions(w):
    """World positions [count, 64, 3] of the Morton-ordered nodes (tests/test_pipeline.py:14-25)."""
    codes = w.table.codes
    out = np.empty((len(codes), 64, 3))
    slots = np.arange(64)
    sx = (slots & 1) | ((slots >> 2) & 2)
    sy = ((slots >> 1) & 1) | ((slots >> 3) & 2)
    sz = ((slots >> 2) & 1) | ((slots >> 4) & 2)
    for b, code in enumerate(codes):
        bx, by, bz = O.decode(int(code))
        out[b, :, 0] = (4 * bx + sx - CELL_BIAS) * w.params.dx
        out[b, :, 1] = (4 * by + sy - CELL_BIAS) * w.params.dx
        out[b, :, 2] = (4 * bz + sz - CELL_BIAS) * w.params.dx
    return out


def paint(w, field):
    npos = node_positions(w)
    vel = np.empty((w.table.count, 4, 64))
    vel[:, 0, :] = 1.0
    v = np.apply_along_axis(field, 2, npos)
    vel[:, 1:4, :] = v.transpose(0, 2, 1)
    w.grid.set_vel(vel)


def test_free_zone_violation_rebuild_steps():
    # tests/test_pipeline.py:73-82
    w = _mk([(8.0, 8.0, 8.0)], [(0.0, 0.0, -120.0)],
            params=SimParams(dx=0.5, dt=1e-2, gravity=(0.0, 0.0, 0.0)))
    for s in range(6):
        w.run_step(s)
    assert w.rebuild_steps[:2] == [0, 4]


def test_single_particle_mass_kat():
    # tests/test_pipeline.py:86-93, 399-404
    w = _mk([(4.0, 4.0, 4.0)], params=SimParams(dx=0.5, dt=1e-4, gravity=(0, 0, 0)), mass=2.0)
    w.run_step(0)
    masses = w.grid.raw[0][:, 0, :]
    assert np.isclose(masses.sum(), 2.0, rtol=1e-6)
    assert np.isclose(masses.max(), 2.0 * 0.75 ** 3, rtol=1e-6)
    assert (w.table.count, w.table.n_gblocks) == (27, 1)


def test_conservation_one_substep(rng):
    # tests/test_pipeline.py:95-106: grid mass/momentum == particle mass/momentum (1e-5)
    pos = rng.uniform(6.0, 10.0, (400, 3))
    vel = rng.normal(0, 30, (400, 3))
    w = _mk(pos, vel, params=SimParams(dx=0.5, dt=1e-4), mass=0.25, collect_conservation=True)
    for s in range(3):
        w.run_step(s)
    rows = np.array(w.conservation)
    assert np.abs(rows[:, 4] - rows[:, 0]).max() / rows[:, 0].max() < 1e-5
    scale = np.abs(rows[:, 1:4]).max()
    assert np.abs(rows[:, 5:8] - rows[:, 1:4]).max() / scale < 1e-5


def test_one_cell_group_27_accumulations(rng):
    # tests/test_pipeline.py:108-118
    pos = np.array([4.1, 4.1, 4.1]) + rng.uniform(0.0, 0.04, (20, 3))
    w = _mk(pos, params=SimParams(dx=0.5, dt=1e-4, gravity=(0, 0, 0)))
    w.run_step(0)
    assert w.store.n_groups == 1
    c = w.counters
    assert int(c[O.C_SUBGROUPS]) == 1 and int(c[O.C_ACCUM]) == 27


def test_free_fall_velocity():
    # tests/test_pipeline.py:129-138
    params = SimParams(dx=0.5, dt=2e-3, gravity=(0.0, 0.0, -981.0))
    w = _mk([(8.0, 8.0, 8.0)], [(3.0, 0.0, 0.0)], params=params)
    w.run_step(0)
    d = w.store.data
    assert np.isclose(d[0, 3, 0], 3.0, atol=1e-5)
    assert np.isclose(d[0, 5, 0], -981.0 * params.dt, rtol=1e-5)


def test_zero_mass_nodes_skipped():
    # tests/test_pipeline.py:140-147
    w = _mk([(8.0, 8.0, 8.0)], params=SimParams(dx=0.5, dt=1e-3))
    w.run_step(0)
    vel = w.grid.vel
    zero = vel[:, 0, :] == 0.0
    for ch in range(1, 4):
        assert (vel[:, ch, :][zero] == 0.0).all()


@pytest.mark.parametrize("mode", ["slip", "sticky"])
def test_box_boundary(mode):
    # tests/test_pipeline.py:149-193
    dx = 0.5
    params = SimParams(dx=dx, dt=1e-3, gravity=(0.0, 0.0, 0.0))
    floor_z = 8 * dx
    boundary = BoundaryBox((dx, dx, floor_z), (31 * dx, 31 * dx, 31 * dx), mode=mode)
    w = _mk([(8.0, 8.0, floor_z + 0.3 * dx)], [(10.0, 0.0, -50.0)], params=params, boundary=boundary)
    w.run_step(0)
    vel, npos = w.grid.vel, node_positions(w)
    live = vel[:, 0, :] > 0
    below = live & (npos[:, :, 2] <= floor_z)
    above = live & (npos[:, :, 2] > floor_z)
    assert below.any() and above.any()
    assert (vel[:, 3, :][below] == 0.0).all()
    if mode == "slip":
        assert np.allclose(vel[:, 1, :][below], 10.0, atol=1e-4)
    else:
        assert (vel[:, 1, :][below] == 0.0).all() and (vel[:, 2, :][below] == 0.0).all()
    assert np.allclose(vel[:, 3, :][above], -50.0, atol=1e-4)


def test_painted_uniform_field(rng):
    # tests/test_pipeline.py:203-217
    w = _mk(rng.uniform(7.0, 9.0, (50, 3)), params=SimParams(dx=0.5, dt=1e-3, gravity=(0, 0, 0)))
    w.run_step(0)
    u = np.array([3.0, -2.0, 1.0])
    paint(w, lambda p: u)
    w._vel_dt = w.params.dt
    w._run_g2p(1)
    d = w.store.data
    mask = d[:, CH_MASS, :] > 0
    for a in range(3):
        assert np.abs(d[:, CH_VEL + a, :][mask] - u[a]).max() < 1e-5
    C = np.stack([d[:, CH_C + k, :][mask] for k in range(9)], axis=-1)
    assert np.abs(C).max() < 2e-4      # fp32: sum of w * v * dpos cancels to ~1e-6 * 4/dx^2


def test_painted_zero_field_keeps_particles_static(rng):
    # tests/test_pipeline.py:219-226
    w = _mk(rng.uniform(7.0, 9.0, (50, 3)), params=SimParams(dx=0.5, dt=1e-3, gravity=(0, 0, 0)))
    w.run_step(0)
    before, _ = w.store.positions_with_ids()
    paint(w, lambda p: np.zeros(3))
    w._run_g2p(1)
    after, _ = w.store.positions_with_ids()
    assert np.array_equal(before, after)


def test_painted_linear_field_recovers_gradient(rng):
    # tests/test_pipeline.py:228-236
    w = _mk(rng.uniform(7.0, 9.0, (50, 3)), params=SimParams(dx=0.5, dt=1e-3, gravity=(0, 0, 0)))
    w.run_step(0)
    A = np.array([[2.0, 1.0, 0.0], [0.5, -1.0, 0.3], [0.0, 0.2, 0.8]])
    paint(w, lambda p: A @ p)
    w._run_g2p(1)
    d = w.store.data
    mask = d[:, CH_MASS, :] > 0
    C = np.stack([d[:, CH_C + k, :][mask] for k in range(9)], axis=-1)
    assert np.abs(C - A.reshape(9)).max() / np.abs(A).max() < 1e-4


def test_quarantine_and_drop_at_rebuild():
    # tests/test_pipeline.py:371-395
    pos = np.array([(8.0, 8.0, 8.0), (9.0, 9.0, 9.0)])
    w = _mk(pos, params=SimParams(dx=0.5, dt=1e-4), collect_conservation=True)
    w.run_step(0)
    d = w.store.data
    d[0, CH_VEL, 0] = np.nan
    w.store.set_data(d)
    w.run_step(1)
    assert int(w.counters[O.C_QUARANTINE]) == 1
    w.run_step(2)
    pm, gm = w.conservation[-1][0], w.conservation[-1][4]
    assert np.isclose(pm, gm, rtol=1e-6)
    p, ids = w.store.positions_with_ids()
    assert len(ids) == 2                      # quarantined particles are still reported
    w.flags.rebuild_needed = True
    w.run_step(3)
    assert w.store.count == 1


def test_stationary_particles_touch_identical_sets(rng):
    # tests/test_pipeline.py:406-416
    w = _mk(rng.uniform(6.0, 10.0, (50, 3)), params=SimParams(dx=0.5, dt=1e-4, gravity=(0, 0, 0)))
    w.run_step(0)
    first = set(w.table.touched_indices(0))
    w.run_step(1)
    w.run_step(2)
    assert set(w.table.touched_indices(0)) == first
    assert first <= set(range(w.table.count))


def test_empty_world_steps_are_noops():
    # tests/test_pipeline.py:418-423
    w = _mk(np.zeros((0, 3)))
    for s in range(3):
        w.run_step(s)
    assert w.table.count == 0 and w.store.count == 0
    assert w.runtime.generations == 3       # tests/test_pipeline.py:425-430


def test_out_of_domain_particle_raises():
    # particles.py:54-57
    w = _mk([(8.0, 8.0, 8.0), (-1.0e9, 0.0, 0.0)])
    with pytest.raises(SpatialDomainError):
        w.run_step(0)


def test_block_touching_domain_boundary_raises():
    # grid.py:372-377: a gblock at block coordinate 0 has no room for its halo
    dx = 0.5
    w = _mk([((-CELL_BIAS + 1.2) * dx,) * 3], params=SimParams(dx=dx, dt=1e-4))
    with pytest.raises(SpatialDomainError):
        w.run_step(0)


def test_append_particles_forces_rebuild_and_mode_conflict(rng):
    # pipeline.py:837-850
    w = _mk(rng.uniform(7.0, 9.0, (40, 3)), params=SimParams(dx=0.5, dt=1e-4), transfer="g2p2g")
    w.run_step(0)
    w.run_step(1)
    assert w.flags.fused_mode
    with pytest.raises(ModeConflictError):
        w.append_particles(rng.uniform(7.0, 9.0, (5, 3)), np.zeros((5, 3)), 1.0)
    w2 = _mk(rng.uniform(7.0, 9.0, (40, 3)), params=SimParams(dx=0.5, dt=1e-4))
    w2.run_step(0)
    assert w2.append_particles(rng.uniform(7.0, 9.0, (5, 3)), np.zeros((5, 3)), 1.0) == 5
    w2.run_step(1)
    assert w2.store.count == 45 and w2.rebuild_steps == [0, 1]
    _, ids = w2.store.positions_with_ids()
    assert sorted(ids.tolist()) == list(range(45))


def test_steady_state_allocates_nothing():
    # tests/test_acceptance.py:287-307: reallocations stop once buffers reached size
    from parity_util import block_scene
    dx = 25.0 / 64.0
    pos, vel = block_scene(8, 3, dx)
    w = _mk(pos, vel, params=SimParams(dx=dx, dt=(1 / 48) / 36),
            boundary=BoundaryBox((8 * dx,) * 3, (40 * dx,) * 3), mass=2.0 * dx ** 3 / 8)
    w.run_frame()
    before = w.realloc_count
    w.run_frame()
    w.run_frame()
    assert len(w.rebuild_steps) >= 3
    assert w.realloc_count == before


def test_pinned_tensor_upload_and_zero_copy_readback(rng):
    """The host-buffer entry used by bench.py's e2e leg: pinned torch tensors are uploaded as they
    are and positions come back through the pinned readback buffers."""
    import torch
    pos = rng.uniform(6.0, 10.0, (300, 3)).astype(np.float32)
    vel = rng.normal(0, 10, (300, 3)).astype(np.float32)
    ids = np.arange(300, dtype=np.int64)[::-1].copy()
    params = SimParams(dx=0.5, dt=1e-4)
    wa = _mk(pos.astype(np.float64), vel.astype(np.float64), params=params, mass=0.5)
    wb = _mk(np.zeros((0, 3)), params=params)
    wa.store._staged.clear(); wa.store.staged_count = 0
    wa.seed_particles(pos, vel, 0.5, ids=ids)
    wb.replace_particles(torch.from_numpy(pos).pin_memory(), torch.from_numpy(vel).pin_memory(), 0.5,
                         torch.from_numpy(ids).pin_memory())
    for s in range(3):
        wa.run_step(s)
        wb.run_step(s)
    pa, ia = wa.store.positions_with_ids()
    pb, ib = wb.store.positions_with_ids(dtype=None)
    assert pb.dtype == np.float32 and np.array_equal(ia, ib)
    # same inputs, same kernels; float atomics may reorder sums between two runs
    assert np.allclose(pa, pb, rtol=0, atol=1e-5)
    assert np.allclose(wa.store.data, wb.store.data, rtol=1e-4, atol=1e-4)


def test_status_block_published_to_mapped_host_memory():
    """mpm_status_publish / mpm_host_alias: the read of out_stats after a gather
    (pipeline.py:1102-1104) is a store to pinned host memory by a kernel, in stream order."""
    import ctypes as C
    import torch
    from paper_2111_00699_b200 import _capi
    lib = _capi.lib()
    words = _capi.STATUS_BYTES // 8
    dev = torch.arange(1, 1 + 2 * words, dtype=torch.int64, device="cuda").reshape(2, words)
    host = torch.zeros((2, words), dtype=torch.int64).pin_memory()
    guard = torch.tensor([17], dtype=torch.int32, device="cuda")
    guard_host = torch.zeros(2, dtype=torch.int32).pin_memory()
    alias, galias = lib.mpm_host_alias(host.data_ptr()), lib.mpm_host_alias(guard_host.data_ptr())
    assert alias and galias
    stream = torch.cuda.current_stream().cuda_stream
    _capi.check(lib.mpm_status_publish(dev[1].data_ptr(), alias + _capi.STATUS_BYTES, guard.data_ptr(),
                                       galias + 4, stream))
    torch.cuda.synchronize()
    assert host[0].abs().sum() == 0 and torch.equal(host[1], dev[1].cpu())
    assert guard_host.tolist() == [0, 17]
    # pageable memory has no device alias; inconsistent arguments are rejected
    assert not lib.mpm_host_alias(torch.zeros(8).data_ptr())
    assert lib.mpm_status_publish(None, alias, None, None, stream) == -1
    assert lib.mpm_status_publish(None, None, None, None, stream) == 0


@pytest.mark.parametrize("transfer", ["g2p2g", "split"])
def test_batched_frames_report_every_step(transfer):
    """Frames enqueued from C (status stored by the grid update / the publish kernel, kernels
    chained with programmatic dependent launch) against the same frames stepped one host call
    at a time: same rebuild steps, same max speed per step, same particles."""
    from parity_util import block_scene
    dx = 25.0 / 64.0
    pos, vel = block_scene(8, 3, dx)
    kw = dict(params=SimParams(dx=dx, dt=(1 / 48) / 36), boundary=BoundaryBox((8 * dx,) * 3, (40 * dx,) * 3),
              mass=2.0 * dx ** 3 / 8, transfer=transfer)
    wa, wb = _mk(pos, vel, **kw), _mk(pos, vel, **kw)
    wb.pipelined = False
    vmax = {0: [], 1: []}
    for k, w in enumerate((wa, wb)):
        pub = w.runtime.publish_vmax
        w.runtime.publish_vmax = lambda slot, wid, v, k=k, pub=pub: (vmax[k].append(v), pub(slot, wid, v))[1]
    for _ in range(3):
        wa.run_frame()
        wb.run_frame()
    assert wa.kernel_calls < wb.kernel_calls          # wa really went through mpm_enqueue_steps
    assert wa.rebuild_steps == wb.rebuild_steps, (wa.rebuild_steps, wb.rebuild_steps)
    assert len(wa.rebuild_steps) >= 3, wa.rebuild_steps
    assert len(vmax[0]) == len(vmax[1])
    assert np.allclose(vmax[0], vmax[1], rtol=1e-4, atol=1e-6)
    pa, ia = wa.store.positions_with_ids()
    pb, ib = wb.store.positions_with_ids()
    assert np.array_equal(ia, ib) and np.allclose(pa, pb, rtol=0, atol=2e-5)


def test_asynchronous_snapshot_readback(rng):
    """positions_with_ids_async: same snapshot as the blocking call, two readbacks in flight."""
    pos = rng.uniform(6.0, 10.0, (500, 3))
    vel = rng.normal(0, 10, (500, 3))
    w = _mk(pos, vel, params=SimParams(dx=0.5, dt=1e-4), mass=0.5)
    handles, expect = [], []
    for s in range(3):
        w.run_step(s)
        handles.append(w.store.positions_with_ids_async())
        if s < 2:
            continue                     # first two handles are left pending over the next steps
    expect = w.store.positions_with_ids(dtype=None)
    p2, i2 = handles[2].wait()
    assert np.array_equal(i2, expect[1]) and np.array_equal(p2, expect[0])
    p1, i1 = handles[1].wait()           # the other buffer pair: the state one step earlier
    assert np.array_equal(np.sort(i1), np.sort(i2)) and not np.array_equal(p1, p2)
