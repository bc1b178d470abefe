"""GPU bring-up: run the CUDA worker next to the oracle / golden dumps and print errors."""
import os, sys, time, traceback
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
from conftest import elastic_setup, fluid_setup, golden
import parity_util as U
from oracle import build as obuild
obuild.build()


def section(name):
    print(f"\n=== {name} ===", flush=True)


def run_case(name, setup, steps=24, **opts):
    section(f"{name} {opts}")
    g = golden(name)
    material, params, boundary = setup
    pos, vel, mass = g["pos"], g["vel"], float(g["mass"])
    wc = U.cuda_worker(pos, vel, mass, material, params, boundary, **opts)
    wo = U.oracle_worker(pos, vel, mass, material, params, boundary, **opts)
    edge = float(pos.max() - pos.min())
    ndef = 1 if int(material.kind) == 0 else 9
    wc.run_step(0); wo.run_step(0)
    if "s0_codes" in g.files:
        print("structure mismatches vs golden:", U.structure_mismatches(wc, g))
    print("perm equal:", np.array_equal(wc.last_perm.cpu().numpy(), wo.last_perm),
          "gidx equal:", np.array_equal(wc.last_gidx.cpu().numpy(), wo.last_gidx))
    print("counts cuda", wc.table.count, wc.table.n_gblocks, wc.store.n_groups, wc.store.count,
          "oracle", wo.table.count, wo.table.n_gblocks, wo.store.n_groups, wo.store.count)
    print("raw0 rel err per channel:", U.grid_errors(wc.grid.raw[0], wo.grid.raw[0]))
    print("vel  rel err per channel:", U.grid_errors(wc.grid.vel, wo.grid.vel))
    print("touched0 equal:", np.array_equal(wc.table.touched[0], wo.table.touched[0][:wo.table.count]))
    sc, so = U.state_by_id(wc), U.state_by_id(wo)
    print("step1 particle errs (x/edge, v rel, F abs, C rel):", U.particle_errors(sc, so, edge, ndef))
    print("counters cuda", wc.counters, "oracle", wo.counters)
    for s in range(1, steps):
        wc.run_step(s); wo.run_step(s)
        if s in (1, 5, 11, steps - 1):
            sc, so = U.state_by_id(wc), U.state_by_id(wo)
            print(f"step {s+1} particle errs:", U.particle_errors(sc, so, edge, ndef),
                  "rebuilds", wc.rebuild_steps, wo.rebuild_steps)
    if wc._pending_gather:
        wc._flush_gather(); wo._flush_gather()
        sc, so = U.state_by_id(wc), U.state_by_id(wo)
        print("flushed particle errs:", U.particle_errors(sc, so, edge, ndef))
    print("mass", wc.store.total_mass(), wo.store.total_mass(), "mom", wc.store.total_momentum(), wo.store.total_momentum())
    print("counters cuda", wc.counters, "oracle", wo.counters)


def guarded(fn, *a, **k):
    try:
        fn(*a, **k)
    except Exception:
        traceback.print_exc()


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0))
    guarded(run_case, "elastic.npz", elastic_setup())
    guarded(run_case, "fluid.npz", fluid_setup())
    guarded(run_case, "fused.npz", elastic_setup(), transfer="g2p2g")
    guarded(run_case, "flip.npz", elastic_setup(flip_blend=0.8), steps=6)
    # timing of a bigger block
    section("timing 1M")
    from paper_2111_00699_b200 import Material, SimParams, BoundaryBox
    dx = 25.0 / 64.0
    pos, vel = U.block_scene(50, 7, dx, origin_cells=(16, 16, 16))
    print("particles", len(pos))
    material = Material.fixed_corotated(2.0, 1.0e5, 0.3)
    params = SimParams(dx=dx, dt=(1 / 48) / 36)
    boundary = BoundaryBox((8 * dx,) * 3, (120 * dx,) * 3)
    for transfer, thr in (("split", 100000), ("g2p2g", 1 << 40)):
        w = U.cuda_worker(pos, vel, 2.0 * dx ** 3 / 8, material, params, boundary,
                          worker_kw=dict(count_stats=False), transfer=transfer, fused_threshold=thr)
        for s in range(4):
            w.run_step(s)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for s in range(4, 40):
            w.run_step(s)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(transfer, "ms/step", (t1 - t0) / 36 * 1e3, "Mpss/s", len(pos) * 36 / (t1 - t0) / 1e6,
              "rebuilds", w.rebuild_steps, "groups", w.store.n_groups, "pblocks", w.table.count)
