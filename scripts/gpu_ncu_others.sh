#!/bin/bash
# full ncu capture of one launch each of the other kernels of the step (1.37 M snow scene):
#   gpurun -- bash scripts/gpu_ncu_others.sh <tag>
tag=$1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" -s $3 -c 1 -f -o gpurun_out/${tag}_$1 \
    python bench.py --scene snow --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
}
cap g2p 'transfer_kernel<\(int\)[0-9], \(bool\)1, \(bool\)0' 3
cap p2g 'transfer_kernel<\(int\)[0-9], \(bool\)0, \(bool\)1' 3
cap grid 'grid_update_kernel' 100
cap sortscatter 'scatter_sorted_kernel' 3
ls -la gpurun_out/${tag}_*
