#!/bin/bash
for f in 0 1; do
  PHJ_PHI_FP32=$f timeout 300 python scripts/transport_act_ab.py 2>/dev/null | head -1 | sed "s/^{/{\"phi_fp32\": $f, /" >> gpurun_out/r2v_transport_ab.jsonl
done
timeout 600 python -m pytest tests/test_gpu_async.py tests/test_gpu_configs.py -q -x > gpurun_out/r2v_tests.log 2>&1; echo "tests rc=$?"
