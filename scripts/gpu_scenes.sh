#!/bin/bash
# one bench line per scene of BASELINE.json's configs (value leg only): gpurun -- bash scripts/gpu_scenes.sh
for spec in "snow" "snow_fc" "sand64k" "sand64k --transfer split" "sand389k" "sand10m --steps 6" "mixed4m --steps 8" "mixed32m --steps 4 --warmup 3" "fountain --steps 8"; do
  set -- $spec
  python bench.py --scene "$@" --no-cpu-baseline --no-e2e > gpurun_out/scene.log 2>&1
  python - "$spec" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/scene.log").read().strip().splitlines()[-1]); r = d.get("roofline") or {}
    print("%-28s frame %8.3f ms  value %7.0f M pss/s  kernel %s ms  frac %s  particles %s" % (
        sys.argv[1], d["ms_per_step"], d["value"], r.get("avg_launch_ms"), r.get("frac"), d["config"].get("particles")))
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/scene.log").read()[-600:])
PY
done
