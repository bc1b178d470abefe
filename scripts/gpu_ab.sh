#!/bin/bash
# A/B of kernel build variants ON the GPU box (variants/ does not travel): each spec is
# "name -DFLAG=.. ..." ; builds paper_2111_00699_b200/variants/libmpm_<name>.so there and times the
# fused kernel of the 1.37 M scene (snow + fixed-corotated) with it.
#   gpurun -- bash scripts/gpu_ab.sh "base -DMPM_MASSFOLD=0" "mf -DMPM_MASSFOLD=1" ...
# SCENES="snow snow_fc" STEPS=10 by default; the in-tree library is timed as "tree".
mkdir -p gpurun_out
SCENES=${SCENES:-"snow snow_fc"}
STEPS=${STEPS:-10}
run_one() {   # name, lib path ("" = in tree)
  for scene in $SCENES; do
    MPM_B200_LIB=$2 python bench.py --scene $scene --steps $STEPS --warmup 3 --no-cpu-baseline --no-e2e --no-pinned-variant \
        > gpurun_out/ab_$1_$scene.log 2> gpurun_out/ab_$1_$scene.err
    python - "$1" "$scene" <<'PY'
import json, sys
name, scene = sys.argv[1:3]
try:
    d = json.loads(open(f"gpurun_out/ab_{name}_{scene}.log").read().strip().splitlines()[-1])
    r = d["roofline"]
    print("%-10s %-8s frame %7.3f ms  value %6.0f  kernel %.4f ms  frac %.4f  share %.3f" % (
        name, scene, d["ms_per_step"], d["value"], r["avg_launch_ms"], r["frac"], r["kernel_share_of_step"]), flush=True)
except Exception as e:
    print(name, scene, "FAILED", e, open(f"gpurun_out/ab_{name}_{scene}.err").read()[-600:])
PY
  done
}
if [ -z "$NOTREE" ]; then MPM_B200_LIB= run_one tree "$PWD/paper_2111_00699_b200/libmpm_b200.so"; fi
for spec in "$@"; do
  set -- $spec
  name=$1; shift
  bash scripts/build_variant.sh $name "$@" > gpurun_out/ab_build_$name.log 2>&1
  run_one $name "$PWD/paper_2111_00699_b200/variants/libmpm_$name.so"
done
