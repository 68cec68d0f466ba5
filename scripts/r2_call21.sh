#!/bin/bash
# Morton-ordered band rows + atomics-free band schedule: schedule test, kernel times, step split
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bands.py -x -q > gpurun_out/r2u_bands_test.log 2>&1; echo "bands test rc=$?"; tail -3 gpurun_out/r2u_bands_test.log
for c in c5 c3; do
  timeout 400 python scripts/band_ab.py $c >> gpurun_out/r2u_morton_ab.jsonl 2>> gpurun_out/r2u_morton_ab.err
done
cat gpurun_out/r2u_morton_ab.jsonl
timeout 600 python scripts/step_breakdown.py c5 float64 > gpurun_out/r2u_step_breakdown.jsonl 2> gpurun_out/r2u_step_breakdown.err; echo "breakdown rc=$?"
tail -1 gpurun_out/r2u_step_breakdown.jsonl
