"""Two ranks, one process each (launched by torch.distributed.run): DistWorker against the
reference dump of the two-worker run.  Usable on a single GPU: with the gloo backend both
ranks share cuda:0 and the halo rows are staged through host memory.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29517 tests/dist_check.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch
import torch.distributed as dist

import parity_util as U
from conftest import elastic_setup, golden
from paper_2111_00699_b200 import PipelineOptions
from paper_2111_00699_b200.dist import DistRuntime, DistWorker, seed_rank
from paper_2111_00699_b200.peer import PeerDistWorker, PeerRuntime


def main():
    backend = os.environ.get("MPM_DIST_BACKEND", "gloo")
    dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ndev)
    torch.cuda.set_device(dev)
    if os.environ.get("MPM_SCENE", "") == "snow":
        return snow_slabs(rank, world, dev)
    if os.environ.get("MPM_SCENE", "") == "repartition":
        return repartition_check(rank, world, dev)
    if os.environ.get("MPM_SCENE", "") == "mixed":
        return mixed_populations(rank, world, dev)
    if os.environ.get("MPM_SCENE", "") == "soak":
        return soak(rank, world, dev)
    g = golden("two_worker.npz")
    material, params, boundary = elastic_setup()
    transfer = os.environ.get("MPM_TRANSFER", "split")
    halo = os.environ.get("MPM_HALO", "sendrecv")     # sendrecv: DistWorker, peer: PeerDistWorker
    frames = os.environ.get("MPM_MODE", "steps") == "frames"
    vmax0 = float(np.linalg.norm(g["vel"], axis=1).max())
    if frames:
        # 24 steps as two device-paced frames of 12 (rebuilds and rollbacks inside)
        import dataclasses
        params = dataclasses.replace(params, steps_per_frame=12, frame_dt=12 * params.dt)
    if halo == "peer":
        rt = PeerRuntime(dev, initial_vmax=vmax0)
        w = PeerDistWorker(rt, params, material, boundary, PipelineOptions(transfer=transfer), device=dev,
                           wait_timeout_ms=20000, lazy_flush=os.environ.get("MPM_LAZY", "0") == "1")
        w.batch_steps = int(os.environ.get("MPM_PEER_BATCH", "4"))   # 0: one guarded step per host call
    else:
        rt = DistRuntime(dev, initial_vmax=vmax0)
        w = DistWorker(rt, params, material, boundary, PipelineOptions(transfer=transfer), device=dev)
    seed_rank(w, g["pos"], g["vel"], float(g["mass"]))
    if frames:
        w.run_frame()
        w.run_frame()
        return finish(w, g, rank, world, transfer, halo, frames)
    w.run_step(0)
    if world == 2 and transfer == "split":
        bad = U.structure_mismatches(w, g, f"w{rank}_s0_")
        assert bad == [], bad
        for c, e in enumerate(U.grid_errors(w.grid.vel, g[f"w{rank}_s0_vel"])):
            assert e <= U.GRID_RTOL, ("vel", rank, c, e)
    for s in range(1, 24):
        w.run_step(s)
    finish(w, g, rank, world, transfer, halo, frames)


def repartition_check(rank, world, dev):
    """Dynamic re-partitioning (dist.repartition): the two-worker scene seeded with a deliberately bad
    partition -- 70 % of the particles on rank 0, the slabs interleaved -- runs 12 steps, re-cuts the
    slabs (particles migrate with their whole state), runs 12 more.  The union must match the
    reference's 24-step state at the short-run bars (the result does not depend on who owns a
    particle), ids and total mass must be preserved and the counts balanced."""
    import dataclasses
    g = golden("two_worker.npz")
    material, params, boundary = elastic_setup()
    params = dataclasses.replace(params, steps_per_frame=12, frame_dt=12 * params.dt)
    halo = os.environ.get("MPM_HALO", "sendrecv")
    transfer = os.environ.get("MPM_TRANSFER", "split")
    vmax0 = float(np.linalg.norm(g["vel"], axis=1).max())
    if halo == "peer":
        w = PeerDistWorker(PeerRuntime(dev, initial_vmax=vmax0), params, material, boundary,
                           PipelineOptions(transfer=transfer), device=dev, wait_timeout_ms=20000)
    else:
        w = DistWorker(DistRuntime(dev, initial_vmax=vmax0), params, material, boundary,
                       PipelineOptions(transfer=transfer), device=dev)
    n = len(g["pos"])
    rng = np.random.default_rng(5)
    owner = (rng.random(n) > 0.7).astype(np.int64) if world == 2 else rng.integers(0, world, n)
    mine = np.flatnonzero(owner == rank)
    w.seed_particles(g["pos"][mine], g["vel"][mine], float(g["mass"]), ids=mine)
    w.run_frame()
    assert w.repartition(tol=10.0) is None           # within tolerance: nothing moves (still collective)
    rep = w.repartition(force=True)
    assert rep is not None and sum(rep["before"]) == n and sum(rep["after"]) == n, rep
    assert max(rep["after"]) - min(rep["after"]) <= max(0.10 * n, 8), rep   # up to one histogram bin (a lattice plane)
    w.run_frame()
    if w._pending_gather:
        w._flush_gather()
    flat, ids = w.store.state_with_ids()
    parts = [None] * world
    dist.all_gather_object(parts, (flat, ids, list(w.rebuild_steps), rep))
    if rank == 0:
        flat = np.concatenate([p[0] for p in parts])
        ids = np.concatenate([p[1] for p in parts])
        assert np.array_equal(np.sort(ids), np.arange(n)), "ids lost or duplicated by the migration"
        state = flat[np.argsort(ids, kind="stable")]
        assert abs(state[:, 15].sum() - n * float(g["mass"])) <= 1e-6 * n * float(g["mass"])
        edge = float(g["pos"].max() - g["pos"].min())
        ex, ev, ef, ec = U.particle_errors(state, g["state_24"], edge, 9)
        print(f"dist_check repartition world={world} halo={halo} transfer={transfer}: {rep['before']} -> "
              f"{[len(p[1]) for p in parts]} (sent {[p[3]['sent'] for p in parts]}), "
              f"x {ex:.2e} v {ev:.2e} F {ef:.2e} rebuilds {[p[2] for p in parts]}")
        assert [len(p[1]) for p in parts] == rep["after"]
        tolx = 1 if transfer == "split" else 10
        assert ex <= tolx * U.X_RTOL_RUN and ev <= tolx * U.V_RTOL_RUN and ef <= tolx * U.F_ATOL_RUN, (ex, ev, ef)
        print("DIST_CHECK_OK")
    dist.barrier()
    dist.destroy_process_group()


def mixed_populations(rank, world, dev):
    """Material populations over ranks (configs[4]): a small snow + sand scene (sand boxes dropped onto
    snow boxes) as `world` peer-mapped ranks = 2 populations x world/2 slabs, each rank with the
    material of its population; one frame of 30 substeps.  The union is compared with the same
    frame run as two logical workers of ONE process (CudaCluster, one per population)."""
    from paper_2111_00699_b200 import CudaCluster, scenes
    from paper_2111_00699_b200.dist import population_layout, seed_population_rank
    W = scenes.mixed_sparse(l=8, pairs_side=2, domain_cells=64, gap_cells=1)
    f32r = lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)
    for p in W.populations:
        p.positions, p.velocities = f32r(p.positions), f32r(p.velocities)
    transfer = os.environ.get("MPM_TRANSFER", "g2p2g")
    opts = PipelineOptions(transfer=transfer, fused_threshold=1 << 62)
    pop, slab, n_slabs = population_layout(rank, world, len(W.populations))
    w = PeerDistWorker(PeerRuntime(dev, initial_vmax=150.0), W.params, W.populations[pop].material, W.boundary,
                       opts, device=dev, wait_timeout_ms=60000, count_stats=False)
    mine = seed_population_rank(w, W.populations)
    w.run_frame()
    flat, ids = w.store.state_with_ids()
    parts = [None] * world
    dist.all_gather_object(parts, (flat, ids, pop, slab, (w.collective_steps, w.device_paced_steps,
                                                           len(w.rebuild_steps))))
    if rank == 0:
        n = W.n_particles
        flat = np.concatenate([p[0] for p in parts])
        ids = np.concatenate([p[1] for p in parts])
        assert np.array_equal(np.sort(ids), np.arange(n))
        state = flat[np.argsort(ids, kind="stable")]
        cl = CudaCluster(2, W.params, [p.material for p in W.populations], W.boundary, opts, initial_vmax=150.0,
                         device=dev, count_stats=False)
        cl.seed_populations([(p.positions, p.velocities, p.particle_mass) for p in W.populations])
        cl.run_frame()
        ref = cl.state_sorted_by_id()
        shared = len(np.intersect1d(cl.workers[0].table.codes, cl.workers[1].table.codes))
        edge = float(max(p.positions.max() for p in W.populations) - min(p.positions.min() for p in W.populations))
        ex, ev, ef, _ = U.particle_errors(state, ref, edge, 9)
        ej = np.abs(state[:, 25] - ref[:, 25]).max()
        print(f"dist_check mixed world={world} ({n_slabs} slab(s) x 2 populations, {n} particles, {shared} pblocks "
              f"shared by the populations): x {ex:.2e} v {ev:.2e} F {ef:.2e} plastic {ej:.2e} vs one process; "
              f"rank -> (population, slab, collective/device-paced/rebuilds): {[(p[2], p[3], p[4]) for p in parts]}")
        assert shared > 0
        assert ex <= 10 * U.X_RTOL_RUN and ev <= 10 * U.V_RTOL_RUN and ef <= 10 * U.F_ATOL_RUN and \
            ej <= 10 * U.F_ATOL_RUN, (ex, ev, ef, ej)
        print("DIST_CHECK_OK")
    dist.barrier()
    dist.destroy_process_group()


def soak(rank, world, dev):
    """Many device-paced frames over peer-mapped ranks (MPM_FRAMES, default 40) of the small snow + sand
    scene, one re-partition in the middle: invariants only (every id exactly once, mass, finiteness),
    the counters of the speculative pipeline reported."""
    from paper_2111_00699_b200 import scenes
    from paper_2111_00699_b200.dist import population_layout, seed_population_rank
    W = scenes.mixed_sparse(l=8, pairs_side=2, domain_cells=64, gap_cells=1)
    frames = int(os.environ.get("MPM_FRAMES", "40"))
    opts = PipelineOptions(transfer=os.environ.get("MPM_TRANSFER", "g2p2g"), fused_threshold=1 << 62)
    one_pop = world % 2 == 1
    if one_pop:          # odd world: one population, plain slabs (and a re-partition half way)
        pop = W.populations[0]
        w = PeerDistWorker(PeerRuntime(dev, initial_vmax=150.0), W.params, pop.material, W.boundary, opts,
                           device=dev, wait_timeout_ms=60000, count_stats=False, lazy_flush=True)
        seed_rank(w, pop.positions, pop.velocities, pop.particle_mass)
        n, mass = len(pop.positions), pop.particle_mass
    else:
        p, _, _ = population_layout(rank, world, 2)
        w = PeerDistWorker(PeerRuntime(dev, initial_vmax=150.0), W.params, W.populations[p].material, W.boundary,
                           opts, device=dev, wait_timeout_ms=60000, count_stats=False, lazy_flush=True)
        seed_population_rank(w, W.populations)
        n, mass = W.n_particles, None
    for f in range(frames):
        w.run_frame()
        if one_pop and f == frames // 2:
            w.repartition(force=True)
    flat, ids = w.store.state_with_ids()
    parts = [None] * world
    dist.all_gather_object(parts, (flat[:, [0, 1, 2, 15]], ids, (w.collective_steps, w.device_paced_steps,
                                                                  w.speculative_discards, len(w.rebuild_steps))))
    if rank == 0:
        ids = np.concatenate([p[1] for p in parts])
        st = np.concatenate([p[0] for p in parts])
        assert np.array_equal(np.sort(ids), np.arange(n)), "ids lost or duplicated"
        assert np.isfinite(st).all()
        if mass is not None:
            assert abs(st[:, 3].sum() - n * mass) <= 1e-5 * n * mass
        print(f"dist_check soak world={world} frames={frames} ({frames * W.params.steps_per_frame} steps): ids / mass / "
              f"finiteness ok; collective / device-paced / discarded / rebuilds per rank {[p[2] for p in parts]}")
        print("DIST_CHECK_OK")
    dist.barrier()
    dist.destroy_process_group()


def snow_slabs(rank, world, dev):
    """The headline scene (1 372 000 particles, snow plasticity, fused transfer) as `world` peer-mapped
    ranks on ONE GPU: a device-paced frame of 30 substeps per rank slab, the union compared with the
    same frame on a single worker.  Functional (the ranks time-slice the device), with the barrier /
    halo counters of the grid update switched on."""
    from paper_2111_00699_b200 import SharedRuntime, scenes
    from paper_2111_00699_b200.worker import CudaWorker
    W = scenes.snow(plastic=True)
    f32r = lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)
    W.positions, W.velocities = f32r(W.positions), f32r(W.velocities)
    opts = PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62)
    w = PeerDistWorker(PeerRuntime(dev, initial_vmax=150.0), W.params, W.material, W.boundary, opts,
                       device=dev, wait_timeout_ms=60000, count_stats=False)
    w.enable_profile()
    seed_rank(w, W.positions, W.velocities, W.particle_mass)
    w.run_frame()
    flat, ids = w.store.state_with_ids()
    parts = [None] * world
    dist.all_gather_object(parts, (flat, ids, w.profile, (w.collective_steps, w.device_paced_steps,
                                                          w.speculative_discards, len(w.rebuild_steps))))
    if rank == 0:
        flat = np.concatenate([p[0] for p in parts])
        ids = np.concatenate([p[1] for p in parts])
        assert np.array_equal(np.sort(ids), np.arange(len(W.positions)))
        state = flat[np.argsort(ids, kind="stable")]
        ws = CudaWorker(0, SharedRuntime(1, initial_vmax=150.0), W.params, W.material, W.boundary, opts,
                        device=dev, count_stats=False)
        part = U.O.partition_particles(W.positions, 1)[0]
        ws.seed_particles(W.positions[part], W.velocities[part], W.particle_mass, ids=part)
        ws.run_frame()
        ref = U.state_by_id(ws)
        edge = float(W.positions.max() - W.positions.min())
        ex, ev, ef, _ = U.particle_errors(state, ref, edge, 9)
        ej = np.abs(state[:, 25] - ref[:, 25]).max()
        print(f"snow_slabs world={world}: x {ex:.2e} v {ev:.2e} F {ef:.2e} J_P {ej:.2e} vs one worker")
        for r, p in enumerate(parts):
            print(f"  rank {r}: {len(p[1])} particles, collective / device-paced / discarded / rebuilds {p[3]}, "
                  f"profile {p[2]}")
        assert ex <= U.X_RTOL_RUN and ev <= U.V_RTOL_RUN and ef <= U.F_ATOL_RUN and ej <= U.F_ATOL_RUN
        assert all(p[2]["grid_updates"] >= 30 and p[2]["halo_bytes_per_step"] > 0 for p in parts)
        print("DIST_CHECK_OK")
    dist.barrier()
    dist.destroy_process_group()


def finish(w, g, rank, world, transfer, halo, frames):
    if w._pending_gather:
        w._flush_gather()
    flat, ids = w.store.state_with_ids()
    # collect everything on rank 0
    parts = [None] * world
    moved = int(w.halo_rows_sent) if halo != "peer" else \
        int(w.device_paced_steps if frames else w.collective_steps)
    dist.all_gather_object(parts, (flat, ids, list(w.rebuild_steps), moved))
    if rank == 0:
        flat = np.concatenate([p[0] for p in parts])
        ids = np.concatenate([p[1] for p in parts])
        state = flat[np.argsort(ids, kind="stable")]
        edge = float(g["pos"].max() - g["pos"].min())
        ex, ev, ef, ec = U.particle_errors(state, g["state_24"], edge, 9)
        print(f"dist_check world={world} transfer={transfer} halo={halo} frames={frames} "
              f"x {ex:.2e} v {ev:.2e} F {ef:.2e} "
              f"rebuilds {[p[2] for p in parts]} halo_rows/steps {[p[3] for p in parts]}")
        if halo == "peer":
            print("peer: collective steps", w.collective_steps, "device-paced", w.device_paced_steps,
                  "of which enqueued from C", w.batched_steps, "discarded", w.speculative_discards)
        if transfer == "split":
            assert ex <= U.X_RTOL_RUN and ev <= U.V_RTOL_RUN and ef <= U.F_ATOL_RUN, (ex, ev, ef)
            if world == 2:
                assert parts[0][2] == list(g["rebuild_steps0"]) and parts[1][2] == list(g["rebuild_steps1"])
        else:
            assert ex <= 10 * U.X_RTOL_RUN and ev <= 10 * U.V_RTOL_RUN, (ex, ev)
        assert all(p[3] > 0 for p in parts)
        print("DIST_CHECK_OK")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
