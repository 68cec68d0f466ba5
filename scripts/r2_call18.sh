#!/bin/bash
for v in 0 1; do
  PHJ_NO_CWT=$v timeout 300 python scripts/band_ab.py c5 | sed "s/^{/{\"no_cwt\": $v, /" >> gpurun_out/r2r_cwt_ab.jsonl 2>> gpurun_out/r2r_cwt_ab.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/r2r_tests.log 2>&1; echo "tests rc=$?"
