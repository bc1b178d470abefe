import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime, partition_particles
from paper_2111_00699_b200.worker import CudaWorker
W = bench.build_world("snow")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
part = partition_particles(W.positions, N)[0]
w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
               PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False, fuse_clear=True, lazy_flush=True)
w.seed_particles(W.positions[part].astype(np.float32), W.velocities[part].astype(np.float32), W.particle_mass, ids=part)
for _ in range(12):
    w.run_frame()
K = 30
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0 = len(w.rebuild_steps)
    e0.record()
    for _ in range(K):
        w.run_frame()
    e1.record(); torch.cuda.synchronize()
    print("slab 1 of %d: %.3f ms/frame (events), rebuilds %d, graph replays %d, env graph=%s" % (N, e0.elapsed_time(e1) / K, len(w.rebuild_steps) - r0, w.rebuild_graph_replays, os.environ.get("MPM_REBUILD_GRAPH", "1")))
