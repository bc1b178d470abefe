#!/bin/bash
# quick GPU check of a kernel change: parity tests, then fused-kernel timings of the 1.37 M scene
# (fixed-corotated and snow).  usage: gpurun -- bash scripts/gpu_quick.sh <tag> [notest]
tag=${1:-quick}
mkdir -p gpurun_out
if [ "$2" != "notest" ]; then
  python -m pytest tests -m gpu -x -q 2>&1 | tail -12 > gpurun_out/${tag}_pytest.log
fi
for scene in snow_fc snow; do
  python bench.py --scene $scene --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_${scene}.log 2>&1
done
python - <<PY
import json
for scene in ("snow_fc", "snow"):
    try:
        d = json.loads(open("gpurun_out/${tag}_%s.log" % scene).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(scene, "value", d["value"], "ms/frame", d["ms_per_step"], "kernel ms", r["avg_launch_ms"], "frac", r["frac"], "share", r["kernel_share_of_step"], r["kernel_ms_per_step"])
    except Exception as e:
        print(scene, "FAILED", e)
PY
cat gpurun_out/${tag}_pytest.log 2>/dev/null | tail -5
