#!/bin/bash
# stencil in the kernel parameters (uniform-register weight operands): parity tests, A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py tests/test_gpu_pruning.py -x -q > gpurun_out/r2ac_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2ac_tests.log
for cs in 0 1; do
  for c in c5 c3; do
    PHJ_CONST_STENCIL=$cs timeout 400 python scripts/band_ab.py $c | sed "s/^{/{\"const_stencil\": $cs, /" >> gpurun_out/r2ac_const_stencil_ab.jsonl 2>> gpurun_out/r2ac_const_stencil_ab.err
  done
done
cat gpurun_out/r2ac_const_stencil_ab.jsonl; tail -3 gpurun_out/r2ac_const_stencil_ab.err
