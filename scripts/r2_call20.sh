#!/bin/bash
for c in c5 c3 c4; do timeout 600 python scripts/profile_step.py $c float64 3 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'config':d['config'],'transport_ms':d['transport_kernel']['kernel_ms'],'phases':d['phases_ms']}))" >> gpurun_out/r2t_tiled_transport.jsonl; done
timeout 1200 python -m pytest tests/test_gpu_async.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x > gpurun_out/r2t_tests.log 2>&1; echo "tests rc=$?"
PHJ_CERT_LOG=gpurun_out/r2t_cert.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k "c3 or c4 or c5_fp64" > gpurun_out/r2t_cert.log 2>&1; echo "cert rc=$?"
