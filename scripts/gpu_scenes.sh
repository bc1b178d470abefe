#!/bin/bash
# One FULL bench JSON line per scene of BASELINE.json's configs (value leg; clocks, roofline and config
# included), appended to gpurun_out/${OUT:-scenes.jsonl}, plus a one-line digest per scene on stdout.
#   gpurun -- bash scripts/gpu_scenes.sh         then copy gpurun_out/scenes.jsonl to profiles/rN_scenes.jsonl
OUT=gpurun_out/${OUT:-scenes.jsonl}
: > "$OUT"
for spec in "snow" "sand64k" "sand64k --transfer split" "sand_mini" "sand389k" "sand1m" "sand10m --steps 6" \
            "mixed4m --steps 8" "mixed32m --steps 4 --warmup 3" "fountain" "fountain --host-paced"; do
  set -- $spec
  python bench.py --scene "$@" --no-cpu-baseline --no-e2e > gpurun_out/scene.log 2> gpurun_out/scene.err
  python - "$spec" "$OUT" <<'PY'
import json, sys
spec, out = sys.argv[1], sys.argv[2]
try:
    line = open("gpurun_out/scene.log").read().strip().splitlines()[-1]
    d = json.loads(line)
    d["bench_args"] = spec
    open(out, "a").write(json.dumps(d) + "\n")
    r, c = d.get("roofline") or {}, d.get("clocks") or {}
    print("%-28s frame %8.3f ms  value %7.0f M pss/s  kernel %s ms  frac %s  particles %s  sm %s MHz %s" % (
        spec, d["ms_per_step"], d["value"], r.get("avg_launch_ms"), r.get("frac"),
        d["config"].get("particles", d["config"].get("particles_max")), c.get("sm_mhz"), c.get("reasons")))
except Exception as e:
    print(spec, "FAILED", e, open("gpurun_out/scene.log").read()[-400:], open("gpurun_out/scene.err").read()[-800:])
PY
done
