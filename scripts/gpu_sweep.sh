#!/bin/bash
# time the fused kernel of several library variants: gpurun -- bash scripts/gpu_sweep.sh <name> ...
for name in "$@"; do
  lib=paper_2111_00699_b200/variants/libmpm_$name.so
  [ "$name" = "default" ] && lib=paper_2111_00699_b200/libmpm_b200.so
  for scene in snow_fc snow; do
    MPM_B200_LIB=$PWD/$lib python bench.py --scene $scene --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_${name}_${scene}.log 2>&1
    python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/sweep_${name}_${scene}.log").read().strip().splitlines()[-1]); r = d["roofline"]
    print("%-14s %-8s kernel %.4f ms  frame %.3f ms  value %.0f" % ("${name}", "${scene}", r["avg_launch_ms"], d["ms_per_step"], d["value"]))
except Exception as e:
    print("${name} ${scene} FAILED", e)
PY
  done
done
