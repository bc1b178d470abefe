import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime, worker as Wm
from paper_2111_00699_b200.worker import CudaWorker
scene = sys.argv[1] if len(sys.argv) > 1 else "sand64k"
W = bench.build_world(scene)
n = len(W.positions)
w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
               PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False,
               fuse_clear=True, lazy_flush=True)
w.seed_particles(W.positions.astype(np.float32), W.velocities.astype(np.float32), W.particle_mass, ids=np.arange(n))
for _ in range(4):
    w.run_frame()
T = {"rebuild_call": 0.0, "wait_call": 0.0, "n": 0, "total": 0.0, "flush": 0.0}
lib = w.lib
orig_rebuild, orig_wait = lib.mpm_rebuild, lib.mpm_rebuild_wait
class L:
    def __getattr__(self, k): return getattr(lib, k)
    def mpm_rebuild(self, *a):
        t = time.perf_counter(); r = orig_rebuild(*a); T["rebuild_call"] += time.perf_counter() - t; return r
    def mpm_rebuild_wait(self, *a):
        t = time.perf_counter(); r = orig_wait(*a); T["wait_call"] += time.perf_counter() - t; return r
w.lib = L()
orig = CudaWorker._rebuild
def timed(self, *a, **k):
    t = time.perf_counter(); r = orig(self, *a, **k); T["total"] += time.perf_counter() - t; T["n"] += 1; return r
CudaWorker._rebuild = timed
of = CudaWorker._flush_gather
def tf(self, *a, **k):
    t = time.perf_counter(); r = of(self, *a, **k); T["flush"] += time.perf_counter() - t; return r
CudaWorker._flush_gather = tf
torch.cuda.synchronize(); t0 = time.perf_counter()
F = 20
for _ in range(F):
    w.run_frame()
torch.cuda.synchronize(); el = time.perf_counter() - t0
k = T["n"]
print(scene, "frames", F, "ms/frame %.3f" % (el / F * 1e3), "rebuilds", k)
print("per rebuild us: _rebuild total %.1f  (mpm_rebuild call %.1f, wait %.1f, python %.1f)  flush call %.1f" % (
    T["total"] / k * 1e6, T["rebuild_call"] / k * 1e6, T["wait_call"] / k * 1e6,
    (T["total"] - T["rebuild_call"] - T["wait_call"]) / k * 1e6, T["flush"] / k * 1e6))
print("graph replays", getattr(w, "rebuild_graph_replays", None), "of", T["n"])
