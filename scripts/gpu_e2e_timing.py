import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime
from paper_2111_00699_b200.worker import CudaWorker
W = bench.build_world("snow")
n = len(W.positions)
pos = torch.from_numpy(W.positions.astype(np.float32)).pin_memory()
vel = torch.from_numpy(W.velocities.astype(np.float32)).pin_memory()
ids = torch.arange(n, dtype=torch.int64).pin_memory()
for lazy in (False, True):
    w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
                   PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False, fuse_clear=True, lazy_flush=lazy)
    for it in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        w.replace_particles(pos, vel, W.particle_mass, ids)
        t1 = time.perf_counter()
        w.run_frame()
        t2 = time.perf_counter()
        p, i = w.store.positions_with_ids(dtype=None)
        t3 = time.perf_counter()
        print("lazy", lazy, "iter", it, "replace %.2f run_frame %.2f readback %.2f ms" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3), "rebuilds", w.frame_rebuilds, "steps", w.frame_steps)
