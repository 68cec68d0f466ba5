#!/bin/bash
PHJ_CERT_LOG=gpurun_out/r2d_cert_full.jsonl timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/r2d_cert_full.log 2>&1; echo "cert rc=$?"
timeout 600 python -m pytest tests/test_gpu_api.py -q > gpurun_out/r2d_api.log 2>&1; echo "api rc=$?"
timeout 900 python scripts/scaling_projection.py c5 float64 > gpurun_out/r2d_scaling_c5.json 2> gpurun_out/r2d_scaling_c5.err; echo "scaling rc=$?"
