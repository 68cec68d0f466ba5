#!/bin/bash
# row-split lane map of the 3D transport: parity tests, kernel times
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py -x -q > gpurun_out/r2z_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2z_tests.log
export PHJ_AB_TRANSPORT_ONLY=1
for c in c5 c3 c4; do
  timeout 400 python scripts/band_ab.py $c >> gpurun_out/r2z_rowsplit_ab.jsonl 2>> gpurun_out/r2z_rowsplit_ab.err
done
cat gpurun_out/r2z_rowsplit_ab.jsonl; tail -3 gpurun_out/r2z_rowsplit_ab.err
