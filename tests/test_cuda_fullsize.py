"""Parity at BASELINE.json's full size (snow scene, 1 372 000 particles): two substeps against the
oracle (the most the CPU does in seconds), then size-independent properties over a whole frame --
sortedness and idempotence of the rebuild, conservation, id preservation, split == fused, one
worker == two workers."""
import numpy as np
import pytest

import parity_util as U

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world():
    from paper_2111_00699_b200 import scenes
    W = scenes.snow(plastic=False)          # the reference-pinned fixed-corotated variant
    f32r = lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)
    W.positions, W.velocities = f32r(W.positions), f32r(W.velocities)
    return W


def _worker(W, **opts):
    return U.cuda_worker(W.positions, W.velocities, W.particle_mass, W.material, W.params, W.boundary,
                         fused_threshold=1 << 62, **opts)


def test_two_substeps_against_the_oracle_at_full_size(world):
    W = world
    assert len(W.positions) == 1372000
    wc = _worker(W, transfer="split")
    wo = U.oracle_worker(W.positions, W.velocities, W.particle_mass, W.material, W.params, W.boundary,
                         transfer="split", fused_threshold=1 << 62)
    for s in range(2):
        wc.run_step(s)
        wo.run_step(s)
    # bit-exact structures
    assert wc.table.n_gblocks == wo.table.n_gblocks and wc.table.count == wo.table.count
    assert np.array_equal(wc.table.codes, wo.table.codes[:wo.table.count])
    assert np.array_equal(wc.table.neighbor, wo.table.neighbor[:wo.table.n_gblocks])
    G = wo.store.n_groups
    assert wc.store.n_groups == G
    assert np.array_equal(wc.store.group_len, wo.store.group_len[:G])
    assert np.array_equal(wc.store.group_block, wo.store.group_block[:G])
    assert np.array_equal(wc.store.orig_id, wo.store.orig_id[:G])
    # fp32 tolerances of parity_util
    edge = float(W.positions.max() - W.positions.min())
    ex, ev, ef, ec = U.particle_errors(U.state_by_id(wc), U.state_by_id(wo), edge, 9)
    print("full size, 2 substeps: x %.2e v %.2e F %.2e C %.2e" % (ex, ev, ef, ec))
    assert ex <= U.X_RTOL and ev <= U.V_RTOL and ef <= U.F_ATOL


def _structure(w):
    st = w.store
    return (w.table.codes.copy(), st.group_len.copy(), st.group_block.copy(), st.orig_id.copy(),
            st.lane_key.copy())


def test_rebuild_is_sorted_and_idempotent_at_full_size(world):
    W = world
    w = _worker(W, transfer="split")
    w.run_step(0)                      # particles have moved: the next rebuild really re-sorts
    w.dt = 0.0
    w._rebuild(1, 1)
    codes, glen, gblock, ids, key = _structure(w)
    assert glen.min() >= 1 and glen.max() <= 32 and int(glen.sum()) == 1372000
    assert (np.diff(gblock) >= 0).all()                      # groups ordered by block
    full = glen == 32
    last_of_block = np.r_[gblock[1:] != gblock[:-1], True]
    assert (full | last_of_block).all()                      # only a block's last group is partial
    live = np.arange(32)[None, :] < glen[:, None]
    assert np.array_equal(np.sort(ids[live]), np.arange(1372000))   # a permutation of the input
    # sortedness: inside a block the particles of one cell are contiguous, i.e. every
    # (block, cell key) pair forms exactly ONE run of lanes
    kflat, bflat = key[live], np.repeat(gblock, glen)
    change = np.r_[True, (kflat[1:] != kflat[:-1]) | (bflat[1:] != bflat[:-1])]
    runs = np.stack([bflat[change], kflat[change]], axis=1)
    # (the sort cell comes from pos / dx, particles.py:53, the lane key from pos * (1 / dx),
    # particles.py:246: the two floors differ for a few particles in a million that sit on a cell
    # face -- as in the reference)
    assert len(runs) - len(np.unique(runs, axis=0)) <= 1e-4 * len(runs)
    # idempotence: rebuilding the unmoved store reproduces table, groups, ids and keys bit for bit
    w._rebuild(2, 0)
    for a, b in zip(_structure(w), (codes, glen, gblock, ids, key)):
        assert np.array_equal(a, b)


def test_frame_properties_at_full_size(world):
    W = world
    wf = _worker(W, transfer="g2p2g")
    ws = _worker(W, transfer="split")
    m0 = wf.store.total_mass() if wf.store.count else None
    wf.run_frame()
    ws.run_frame()
    assert wf._global_step == ws._global_step == W.params.steps_per_frame
    n, mass = 1372000, W.particle_mass
    assert wf.store.total_mass() == pytest.approx(n * mass, rel=1e-6)        # mass conserved
    pos_f, ids_f = wf.store.positions_with_ids()
    assert np.array_equal(np.sort(ids_f), np.arange(n))                       # ids preserved
    assert np.isfinite(pos_f).all() and int(wf.counters[1]) == 0              # nothing quarantined
    lo = np.asarray(W.boundary.min_corner) - 1e-3
    hi = np.asarray(W.boundary.max_corner) + 1e-3
    assert (pos_f >= lo).all() and (pos_f <= hi).all()                        # slip box holds
    # momentum: horizontal components stay ~0 (symmetric drop), vertical = gravity + floor impulse < 0
    p = wf.store.total_momentum()
    pz_free = n * mass * (-150.0 - 981.0 * W.params.frame_dt)
    assert abs(p[0]) <= 1e-3 * abs(pz_free) and abs(p[1]) <= 1e-3 * abs(pz_free)
    assert pz_free * 1.0001 <= p[2] < 0.0
    # fused G2P2G == split P2G + G2P (pipeline.py:604-653) and same rebuild cadence
    sf, ss = U.state_by_id(wf), U.state_by_id(ws)
    edge = float(W.positions.max() - W.positions.min())
    ex, ev, ef, _ = U.particle_errors(sf, ss, edge, 9)
    print("full size frame, fused vs split: x %.2e v %.2e F %.2e" % (ex, ev, ef), wf.rebuild_steps)
    assert ex <= U.X_RTOL_RUN and ev <= U.V_RTOL_RUN and ef <= U.F_ATOL_RUN
    assert wf.rebuild_steps == ws.rebuild_steps


def test_two_workers_equal_one_at_full_size(world):
    from paper_2111_00699_b200 import CudaCluster, PipelineOptions
    W = world
    states = []
    for nw in (1, 2):
        cl = CudaCluster(nw, W.params, W.material, W.boundary,
                         PipelineOptions(transfer="split", fused_threshold=1 << 62), initial_vmax=150.0)
        cl.seed(W.positions, W.velocities, W.particle_mass)
        for s in range(6):
            cl.run_step(s)
        states.append(cl.state_sorted_by_id())
    edge = float(W.positions.max() - W.positions.min())
    ex, ev, ef, _ = U.particle_errors(states[1], states[0], edge, 9)
    print("full size, 2 workers vs 1: x %.2e v %.2e F %.2e" % (ex, ev, ef))
    assert ex <= U.X_RTOL_RUN and ev <= U.V_RTOL_RUN and ef <= U.F_ATOL_RUN
