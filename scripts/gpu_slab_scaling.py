"""Upper bound of the strong-scaling efficiency from ONE GPU: the frame time of one rank's slab of
the 1.37 M snow scene (1/N of the particles, the reference's partition) run alone -- everything a
rank does except waiting for its peers and adding their halo rows.  e_max(N) = T(1) / (N T_slab(N)).

    python scripts/gpu_slab_scaling.py          (on a GPU box)
"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime, partition_particles
from paper_2111_00699_b200.worker import CudaWorker

W = bench.build_world(sys.argv[1] if len(sys.argv) > 1 else "snow")
n = len(W.positions)
t1 = None
for N in (1, 2, 4, 8):
    worst = 0.0
    for r in sorted({0, N // 2, N - 1}):
        part = partition_particles(W.positions, N)[r]
        w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
                       PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False,
                       fuse_clear=True, lazy_flush=True)
        w.seed_particles(W.positions[part].astype(np.float32), W.velocities[part].astype(np.float32),
                         W.particle_mass, ids=part)
        for _ in range(3):
            w.run_frame()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        K = 10
        for _ in range(K):
            w.run_frame()
        torch.cuda.synchronize()
        worst = max(worst, (time.perf_counter() - t0) / K * 1e3)
        del w
    if N == 1:
        t1 = worst
    print("N=%d  slowest slab %.3f ms/frame (%d particles per rank)  e_max = %.2f  (%.0f fps)"
          % (N, worst, n // N, t1 / (N * worst), 1e3 / worst), flush=True)
