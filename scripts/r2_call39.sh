#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/e2e_breakdown.py c5 2>&1 | tail -8
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_async.py -x -q > gpurun_out/r2ak_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2ak_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c5_fp64 or c3" > gpurun_out/r2ak_cert.log 2>&1; echo "cert rc=$?"; tail -3 gpurun_out/r2ak_cert.log
