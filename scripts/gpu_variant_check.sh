#!/bin/bash
# Build a kernel variant ON the GPU box, run the parity tests with it, time it and (NCU=1) capture it:
#   gpurun -- bash scripts/gpu_variant_check.sh <name> -DFLAG=... ...
#   -> gpurun_out/var_<name>_pytest.log, ab_<name>_<scene>.log, var_<name>_<scene>.ncu-rep
name=$1; shift
mkdir -p gpurun_out
bash scripts/build_variant.sh $name "$@" > gpurun_out/ab_build_$name.log 2>&1
export MPM_B200_LIB=$PWD/paper_2111_00699_b200/variants/libmpm_$name.so
ls -la $MPM_B200_LIB
python -m pytest tests/test_cuda_parity.py tests/test_cuda_pipeline.py tests/test_cuda_fullsize.py -m gpu -x -q 2>&1 | tail -8 | tee gpurun_out/var_${name}_pytest.log
for scene in ${SCENES:-snow_fc snow}; do
  python bench.py --scene $scene --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-pinned-variant > gpurun_out/ab_${name}_$scene.log 2> gpurun_out/ab_${name}_$scene.err
  python - $name $scene <<'PY'
import json, sys
name, scene = sys.argv[1:3]
try:
    d = json.loads(open(f"gpurun_out/ab_{name}_{scene}.log").read().strip().splitlines()[-1]); r = d["roofline"]
    print("%-10s %-8s frame %7.3f ms  value %6.0f  kernel %.4f ms  frac %.4f" % (name, scene, d["ms_per_step"], d["value"], r["avg_launch_ms"], r["frac"]))
except Exception as e:
    print(name, scene, "FAILED", e, open(f"gpurun_out/ab_{name}_{scene}.err").read()[-600:])
PY
  if [ -n "$NCU" ]; then
    ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k 'regex:transfer_kernel<\(int\)[0-9], \(bool\)1, \(bool\)1' -s 100 -c 1 -f -o gpurun_out/var_${name}_${scene} \
      python bench.py --scene $scene --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-pinned-variant > /dev/null 2>&1
  fi
done
