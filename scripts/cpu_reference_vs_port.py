#!/usr/bin/env python
"""Build container only: the REAL reference (numba `mpmbench.bench.run`, imported from
/root/reference) timed next to this repository's C port of it (oracle/) on the same scenes, same
host, one worker thread -- the factor that translates `bench.py`'s `kind: "port"` CPU numbers into
reference numbers (BASELINE.md section 4 plan).

    NUMBA_CACHE_DIR=/tmp/numba_cache python scripts/cpu_reference_vs_port.py [--frames 3]

Writes profiles/r2_cpu_reference_vs_port.json.  The GPU box has no /root/reference: nothing in the
tests or in bench.py runs this."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import numpy as np  # noqa: E402


def time_reference(l, boxes, frames, workers):
    sys.path.insert(0, "/root/reference/pkg/src")
    from mpmbench.bench import RunConfig, run
    run(RunConfig(scene="sand_blocks", l=6, boxes=1, frames=1, workers=workers))     # JIT warm-up
    res = run(RunConfig(scene="sand_blocks", l=l, boxes=boxes, frames=frames, workers=workers))
    ms = [r.ms_total for r in res.rows]
    steady = ms[1:] if len(ms) > 1 else ms
    n = res.particle_count
    return {"particles": n, "ms_per_frame_steady_mean": float(np.mean(steady)),
            "ms_per_frame_steady_min": float(np.min(steady)), "frames": frames,
            "M_pss_per_s": n * 36 / (np.mean(steady) * 1e-3) / 1e6}


def time_port(l, boxes, frames, workers):
    from oracle import build as obuild
    obuild.build()
    from oracle import mpm_oracle as O
    from paper_2111_00699_b200 import PipelineOptions, scenes
    W = scenes.sand_blocks(l=l, boxes=boxes)
    cl = O.OracleCluster(workers, W.params, W.material, W.boundary, PipelineOptions(),
                         initial_vmax=150.0, threads=workers > 1)
    cl.seed(W.positions, W.velocities, W.particle_mass)
    ms = []
    for _ in range(frames):
        t0 = time.perf_counter()
        cl.run_frame()
        ms.append((time.perf_counter() - t0) * 1e3)
    steady = ms[1:] if len(ms) > 1 else ms
    n = len(W.positions)
    return {"particles": n, "ms_per_frame_steady_mean": float(np.mean(steady)),
            "ms_per_frame_steady_min": float(np.min(steady)), "frames": frames,
            "M_pss_per_s": n * 36 / (np.mean(steady) * 1e-3) / 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=3)
    a = ap.parse_args()
    out = {"host": {"cpus": os.cpu_count()}, "rows": []}
    for name, l, boxes in (("sand_blocks l=12 boxes=4 (55 296)", 12, 4), ("sand_blocks l=20 boxes=1 (64 000)", 20, 1)):
        for workers in (1, 4):
            ref = time_reference(l, boxes, a.frames, workers)
            port = time_port(l, boxes, a.frames, workers)
            row = {"scene": name, "workers": workers, "reference_numba": ref, "c_port": port,
                   "port_over_reference": port["M_pss_per_s"] / ref["M_pss_per_s"]}
            print(json.dumps(row), flush=True)
            out["rows"].append(row)
    with open(os.path.join(ROOT, "profiles", "r2_cpu_reference_vs_port.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
