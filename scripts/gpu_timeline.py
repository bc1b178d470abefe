"""GPU timeline of a few frames (CUPTI activity records through torch.profiler; the library's
kernels are launched from C but belong to this process, so they are all seen): busy time per
kernel, idle gaps of the device and what surrounds them.

    python scripts/gpu_timeline.py [scene] [frames] [N rank]     (on a GPU box; N rank = one slab of N)
"""
import collections, json, os, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2111_00699_b200 import PipelineOptions, SharedRuntime
from paper_2111_00699_b200.worker import CudaWorker

scene = sys.argv[1] if len(sys.argv) > 1 else "snow"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
W = bench.build_world(scene)
if len(sys.argv) > 4:
    # one rank's slab of the scene run alone: python scripts/gpu_timeline.py snow 4 8 0
    from paper_2111_00699_b200 import partition_particles
    part = partition_particles(W.positions, int(sys.argv[3]))[int(sys.argv[4])]
    W.positions, W.velocities = W.positions[part], W.velocities[part]
n = len(W.positions)
w = CudaWorker(0, SharedRuntime(1, 150.0), W.params, W.material, W.boundary,
               PipelineOptions(transfer="g2p2g", fused_threshold=1 << 62), count_stats=False,
               fuse_clear=True, lazy_flush=True)
w.seed_particles(W.positions.astype(np.float32), W.velocities.astype(np.float32), W.particle_mass,
                 ids=np.arange(n))
for _ in range(int(os.environ.get("WARM", "4"))):
    w.run_frame()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
r0 = len(w.rebuild_steps)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(frames):
        w.run_frame()
    torch.cuda.synchronize()
path = os.path.join(tempfile.gettempdir(), "mpm_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ks = sorted(((e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
             if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e))
t0, t1 = ks[0][0], max(k[1] for k in ks)
busy = collections.Counter(); cnt = collections.Counter()
for a, b, nme in ks:
    key = nme.split("(")[0][-60:]
    busy[key] += b - a; cnt[key] += 1
span = t1 - t0
tot = sum(busy.values())
print("scene %s: %d frames, %d rebuilds, span %.3f ms = %.3f ms/frame, kernels busy %.3f ms (%.1f %%)"
      % (scene, frames, len(w.rebuild_steps) - r0, span / 1e3, span / 1e3 / frames, tot / 1e3, 100 * tot / span))
for k, t in busy.most_common(14):
    print("   %8.1f us %5.1f %%  x%-5d %s" % (t, 100 * t / span, cnt[k], k))
gaps = []
end = ks[0][1]
prev = ks[0][2]
for a, b, nme in ks[1:]:
    if a > end:
        gaps.append((a - end, prev.split("(")[0][-40:], nme.split("(")[0][-40:]))
    if b > end:
        end, prev = b, nme
print("idle total %.3f ms in %d gaps" % (sum(g[0] for g in gaps) / 1e3, len(gaps)))
agg = collections.Counter(); agc = collections.Counter()
for d, p, q in gaps:
    agg[(p, q)] += d; agc[(p, q)] += 1
for (p, q), d in agg.most_common(16):
    print("   %8.1f us  x%-4d mean %6.1f us   %s -> %s" % (d, agc[(p, q)], d / agc[(p, q)], p, q))
# raw intervals of a stretch of steady steps (RAW=<n> kernels): start / end relative to the first
if os.environ.get("RAW"):
    nraw = int(os.environ["RAW"])
    mid = len(ks) // 2
    # start at a fused transfer kernel (RAW_AT=rebuild: a few kernels before a rebuild instead)
    if os.environ.get("RAW_AT") == "rebuild":
        while mid < len(ks) and "rebuild_init" not in ks[mid][2]:
            mid += 1
        mid = max(mid - 12, 0)
    else:
        while mid < len(ks) and "transfer_kernel" not in ks[mid][2]:
            mid += 1
    base = ks[mid][0]
    prev_end = None
    for a, b, nme in ks[mid:mid + nraw]:
        print("   start %9.1f  end %9.1f  dur %7.1f  gap-from-prev-end %7.1f   %s"
              % (a - base, b - base, b - a, (a - prev_end) if prev_end is not None else 0.0, nme.split("(")[0][-48:]))
        prev_end = b
