"""Where the interpreter's time goes in run_frame (cProfile, sorted by own time).
    python scripts/gpu_host_profile.py [scene] [frames]"""
import cProfile, os, pstats, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime
from paper_2111_00699_b200.worker import CudaWorker
scene = sys.argv[1] if len(sys.argv) > 1 else "sand64k"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 12
W = bench.build_world(scene)
n = len(W.positions)
w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
               PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False,
               fuse_clear=True, lazy_flush=True)
w.seed_particles(W.positions.astype(np.float32), W.velocities.astype(np.float32), W.particle_mass, ids=np.arange(n))
for _ in range(4):
    w.run_frame()
torch.cuda.synchronize()
r0 = len(w.rebuild_steps)
pr = cProfile.Profile()
pr.enable()
for _ in range(frames):
    w.run_frame()
torch.cuda.synchronize()
pr.disable()
print("frames", frames, "rebuilds", len(w.rebuild_steps) - r0)
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
