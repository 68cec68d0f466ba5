#!/bin/bash
# transport gather batch with fewer instructions + non-returning sticky-mask atomics: parity tests, kernel times
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_bands.py -x -q > gpurun_out/r2x_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2x_tests.log
for c in c5 c3; do
  timeout 400 python scripts/band_ab.py $c >> gpurun_out/r2x_transport_ab.jsonl 2>> gpurun_out/r2x_transport_ab.err
done
cat gpurun_out/r2x_transport_ab.jsonl
