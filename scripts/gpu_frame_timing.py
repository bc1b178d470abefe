"""Where a frame's wall time goes on the 1.37 M snow scene: per frame wall, rebuild host wall,
number of rebuilds, kernel event sums."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime
from paper_2111_00699_b200.worker import CudaWorker
W = bench.build_world(sys.argv[1] if len(sys.argv) > 1 else "snow")
n = len(W.positions)
w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
               PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False, fuse_clear=True)
w.seed_particles(W.positions.astype(np.float32), W.velocities.astype(np.float32), W.particle_mass, ids=np.arange(n))
for _ in range(3):
    w.run_frame()
torch.cuda.synchronize()
w.time_kernels = True
rows = []
for f in range(12):
    w.kernel_events.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    w.run_frame()
    torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3
    ph = w.phase_ms
    ksum = sum(a.elapsed_time(b) for _, a, b in w.kernel_events)
    rows.append((wall, ph["rebuild"], w.frame_rebuilds, ksum, w.speculative_discards))
    print("frame %2d wall %.2f ms  rebuild(host) %.2f ms x%d  timed kernels %.2f ms  discards(total) %d" % (f, *rows[-1]))
a = np.array(rows)
print("mean wall %.2f  rebuild %.2f  kernels %.2f  other %.2f" % (a[:,0].mean(), a[:,1].mean(), a[:,3].mean(), (a[:,0]-a[:,1]-a[:,3]).mean()))
