"""Soak: many frames of several scenes through the batched / speculative frame driver, checking after
every block of frames that no particle was lost or duplicated, that mass is conserved, that the
state is finite and that no addressing error was counted.     python scripts/gpu_soak.py [frames]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime
from paper_2111_00699_b200.worker import CudaWorker

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for scene, transfer, graph in (("sand64k", "g2p2g", False), ("sand64k", "split", False), ("sand64k", "g2p2g", True),
                               ("sand389k", "g2p2g", False), ("snow", "g2p2g", False), ("snow_fc", "split", False)):
    W = bench.build_world(scene)
    n = len(W.positions)
    w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
                   PipelineOptions(transfer=transfer, fused_threshold=1 << 62), count_stats=False,
                   fuse_clear=True, lazy_flush=True)
    w.rebuild_graph = graph
    w.seed_particles(W.positions.astype(np.float32), W.velocities.astype(np.float32), W.particle_mass, ids=np.arange(n))
    k = frames if n < 500_000 else max(frames // 4, 20)
    t0 = time.perf_counter()
    for f in range(k):
        w.run_frame()
        if (f + 1) % max(k // 4, 1) == 0:
            pos, ids = w.store.positions_with_ids()
            assert len(ids) == n and np.array_equal(np.sort(ids), np.arange(n)), (scene, f, len(ids))
            assert np.isfinite(pos).all()
            m = w.store.total_mass()
            assert abs(m - n * W.particle_mass) <= 1e-5 * n * W.particle_mass, (scene, f, m)
            w._check_addressing()
    torch.cuda.synchronize()
    print("%-9s %-6s graph=%d  %4d frames ok: %d steps, %d rebuilds (%d replayed), %d speculative steps discarded, "
          "%.2f ms/frame incl. checks" % (scene, transfer, graph, k, w._global_step, len(w.rebuild_steps),
                                          w.rebuild_graph_replays, w.speculative_discards,
                                          (time.perf_counter() - t0) / k * 1e3), flush=True)
    del w
print("SOAK_OK")
