#!/bin/bash
timeout 300 python scripts/band_ab.py c5 > gpurun_out/r2u_screen_ab.jsonl 2> gpurun_out/r2u_screen_ab.err; echo "ab rc=$?"
for c in c5 c3 c2; do timeout 600 python scripts/profile_step.py $c float64 3 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'config':d['config'],'patch_ms':d['patch_kernel']['kernel_ms'],'phases':d['phases_ms']}))" >> gpurun_out/r2u_steps.jsonl; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_async.py tests/test_gpu_pruning.py -q -x > gpurun_out/r2u_tests.log 2>&1; echo "tests rc=$?"
PHJ_CERT_LOG=gpurun_out/r2u_cert.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k "c2_fp64 or c3 or c5_fp64" > gpurun_out/r2u_cert.log 2>&1; echo "cert rc=$?"
