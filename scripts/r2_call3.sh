#!/bin/bash
timeout 600 python scripts/debug_missed.py 129 c3 > gpurun_out/r2c_missed.log 2>&1; echo "debug rc=$?"
PHJ_CERT_LOG=gpurun_out/r2c_cert_full.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -k "c2_fp64 or c2_ref or c3 or c4" > gpurun_out/r2c_cert_full.log 2>&1; echo "cert rc=$?"
timeout 600 python -m pytest tests/test_gpu_api.py -q > gpurun_out/r2c_api.log 2>&1; echo "api rc=$?"
