#!/bin/bash
# full ncu capture of ONE launch of the fused G2P2G kernel (late in the warm-up) per scene:
#   gpurun -- bash scripts/gpu_ncu_full.sh <tag> [scene ...]   -> gpurun_out/<tag>_<scene>.ncu-rep
tag=$1; shift
for s in "${@:-snow_fc snow}"; do
  for scene in $s; do
    ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k 'regex:transfer_kernel<\(int\)[0-9], \(bool\)1, \(bool\)1' -s 100 -c 1 -f -o gpurun_out/${tag}_${scene} \
      python bench.py --scene $scene --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  done
done
ls -la gpurun_out/${tag}_*
