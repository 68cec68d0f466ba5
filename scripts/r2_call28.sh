#!/bin/bash
# swizzled 3D solve tile (conflict-free LDS.64 cell loads): parity tests, kernel times
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py tests/test_gpu_pruning.py -x -q > gpurun_out/r2ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2ab_tests.log
for c in c5 c3; do
  timeout 400 python scripts/band_ab.py $c >> gpurun_out/r2ab_swizzle_ab.jsonl 2>> gpurun_out/r2ab_swizzle_ab.err
done
cat gpurun_out/r2ab_swizzle_ab.jsonl; tail -3 gpurun_out/r2ab_swizzle_ab.err
timeout 300 python scripts/profile_step.py c4 float64 3 2>&1 | tail -1 | cut -c1-600
