"""GPU bring-up of the plastic kinds: CUDA vs the float64 oracle definition."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import parity_util as U
from paper_2111_00699_b200 import BoundaryBox, Material, SimParams
from oracle import build as ob
ob.build()
dx = 25.0 / 64.0
pos, vel = U.block_scene(6, 11, dx, origin_cells=(10, 10, 9), speed=-250.0)
params = SimParams(dx=dx, dt=(1 / 48) / 36)
boundary = BoundaryBox((8 * dx,) * 3, (40 * dx,) * 3, mode="slip")
mass = 2.0 * dx ** 3 / 8
edge = float(pos.max() - pos.min())
for name, mat in (("snow", Material.snow(2.0, 1.0e5, 0.3, hardening=5.0)), ("sand", Material.sand(2.0, 1.0e5, 0.3))):
    for transfer in ("split", "g2p2g"):
        wc = U.cuda_worker(pos, vel, mass, mat, params, boundary, transfer=transfer)
        wo = U.oracle_worker(pos, vel, mass, mat, params, boundary, transfer=transfer)
        for s in range(72):
            wc.run_step(s); wo.run_step(s)
            if s in (0, 1, 11, 35, 71):
                a, b = wc, wo
                if a._pending_gather:
                    pass
                sc, so = U.state_by_id(wc), U.state_by_id(wo)
                ex, ev, ef, ec = U.particle_errors(sc, so, edge, 9)
                ep = np.abs(sc[:, 25] - so[:, 25]).max()
                print(name, transfer, "step", s + 1, "x %.2e v %.2e F %.2e plastic %.2e" % (ex, ev, ef, ep),
                      "plastic range", so[:, 25].min(), so[:, 25].max(), "rebuilds", wc.rebuild_steps, wo.rebuild_steps, flush=True)
        print(name, transfer, "counters", wc.counters, wo.counters)
