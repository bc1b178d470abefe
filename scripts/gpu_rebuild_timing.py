import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime
from paper_2111_00699_b200.worker import CudaWorker
W = bench.build_world(sys.argv[1] if len(sys.argv) > 1 else "snow_fc")
n = len(W.positions)
w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
               PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False, fuse_clear=True)
w.seed_particles(W.positions, W.velocities, W.particle_mass, ids=np.arange(n))
for _ in range(3):
    w.run_frame()
torch.cuda.synchronize()
# time forced rebuilds
orig_call = w._call
acc = {}
def timed_call(name, *args):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    orig_call(name, *args)
    torch.cuda.synchronize(); acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
ts = []
for rep in range(6):
    w.flags.rebuild_needed = True
    step = w._global_step
    torch.cuda.synchronize(); t0 = time.perf_counter()
    w.dt = W.params.dt
    w.run_step(step)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    w.run_step(step + 1); w.run_step(step + 2)
print("rebuild step wall ms:", [round(t * 1e3, 3) for t in ts])
torch.cuda.synchronize(); t0 = time.perf_counter()
for k in range(10):
    w.run_step(w._global_step)
torch.cuda.synchronize(); print("plain sync step ms:", (time.perf_counter() - t0) / 10 * 1e3)
w._call = timed_call
for rep in range(4):
    w.flags.rebuild_needed = True
    w.run_step(w._global_step)
    w.run_step(w._global_step)
print({k: round(v / 4 * 1e3, 3) for k, v in acc.items()})
w._call = orig_call
# pure python overhead of a rebuild: time _rebuild host-side with kernels tiny? report take_staged etc.
import cProfile, pstats
pr = cProfile.Profile()
w.flags.rebuild_needed = True
pr.enable(); w.run_step(w._global_step); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
