#!/bin/bash
# Everything the round's profiles/ entries come from, in one GPU call:
#   gpurun --timeout 3000 -- bash scripts/gpu_round_profile.sh r2f
# -> gpurun_out/<tag>_*: full ncu captures of the fused kernel (snow, snow_fc), the launch list of the
#    bench command, one bench line per scene, the slab-scaling bound, timelines, the multi-rank log.
tag=${1:-rN}
mkdir -p gpurun_out
bash scripts/gpu_ncu_full.sh $tag snow snow_fc > gpurun_out/${tag}_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_snow_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-pinned-variant > gpurun_out/${tag}_launches_bench.log 2>&1
OUT=${tag}_scenes.jsonl bash scripts/gpu_scenes.sh > gpurun_out/${tag}_scenes.txt 2>&1
python scripts/gpu_slab_scaling.py > gpurun_out/${tag}_slab_scaling.txt 2>&1
python scripts/gpu_timeline.py snow 6 > gpurun_out/${tag}_timeline_snow.txt 2>&1
python scripts/gpu_timeline.py snow 6 8 0 > gpurun_out/${tag}_timeline_snow_slab_1_of_8.txt 2>&1
python scripts/gpu_timeline.py sand64k > gpurun_out/${tag}_timeline_sand64k.txt 2>&1
python scripts/gpu_kernel_vs_age.py snow_fc 30 > gpurun_out/${tag}_kernel_vs_age_fc.txt 2>&1
python -m pytest tests/test_cuda_dist.py -m gpu -q -s 2>&1 | grep -E "dist_check|snow_slabs|^  rank|^peer:|passed|failed" > gpurun_out/${tag}_multirank_one_gpu.txt
tail -3 gpurun_out/${tag}_multirank_one_gpu.txt; cat gpurun_out/${tag}_scenes.txt gpurun_out/${tag}_slab_scaling.txt
