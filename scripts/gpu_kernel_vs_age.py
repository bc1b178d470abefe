"""Fused-kernel duration against the number of steps since the last rebuild (lanes are cell-sorted
at a rebuild and drift apart afterwards):   python scripts/gpu_kernel_vs_age.py [scene] [frames]"""
import os, sys, collections
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime
from paper_2111_00699_b200.worker import CudaWorker

scene = sys.argv[1] if len(sys.argv) > 1 else "snow"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40
W = bench.build_world(scene)
n = len(W.positions)
w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
               PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False,
               fuse_clear=True, lazy_flush=True)
w.seed_particles(W.positions.astype(np.float32), W.velocities.astype(np.float32), W.particle_mass, ids=np.arange(n))
for _ in range(3):
    w.run_frame()
w.time_kernels = True
w.kernel_events.clear()
for _ in range(frames):
    w.run_frame()
torch.cuda.synchronize()
by = collections.defaultdict(list)
for name, a, b in w.kernel_events:
    if name == "mpm_g2p2g" and getattr(a, "age", -1) >= 0:
        by[a.age].append(a.elapsed_time(b))
print("scene", scene, "rebuilds", len(w.rebuild_steps), "in", w._global_step, "steps")
for age in sorted(by):
    v = by[age]
    print("age %3d  n %3d  mean %.4f ms  min %.4f  max %.4f" % (age, len(v), np.mean(v), np.min(v), np.max(v)))
allv = [x for v in by.values() for x in v]
print("all: mean %.4f ms over %d samples" % (np.mean(allv), len(allv)))
