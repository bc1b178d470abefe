#!/bin/bash
# a handful of ncu counters of the fused kernel (one launch late in the warm-up) for both
# variants of the 1.37 M scene.  usage: gpurun -- bash scripts/gpu_ncu_light.sh <tag>
tag=${1:-light}
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__thread_inst_executed_per_inst_executed.ratio
for r in barrier branch_resolving dispatch_stall lg_throttle long_scoreboard math_pipe_throttle mio_throttle no_instruction not_selected short_scoreboard wait; do
  M=$M,smsp__average_warps_issue_stalled_${r}_per_issue_active.ratio
done
for scene in snow_fc snow; do
  ncu --metrics $M --clock-control none -k regex:transfer_kernel -s 150 -c 1 --csv --log-file gpurun_out/${tag}_${scene}_ncu.csv \
    python bench.py --scene $scene --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("gpurun_out/${tag}_${scene}_ncu.csv")) if len(r) > 10]
h = rows[0]; iN, iV, iK = h.index("Metric Name"), h.index("Metric Value"), h.index("Kernel Name")
print("${scene}", rows[1][iK][:60])
for r in rows[1:]:
    print("   %-75s %s" % (r[iN].replace("smsp__average_warps_issue_stalled_", "stall "), r[iV]))
PY
done
