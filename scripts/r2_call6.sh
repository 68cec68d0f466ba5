#!/bin/bash
# banded 3D transport: correctness (reduced + full-size certificates) and speed
for c in c3 c4 c5; do
  for b in 0 1; do
    PHJ_TRANSPORT_BANDED=$b timeout 600 python scripts/profile_step.py $c float64 3 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'config':d['config'],'banded':$b,'transport_ms':d['transport_kernel']['kernel_ms'],'phases':d['phases_ms'],'tsweeps':[min(d['transport_sweeps']),max(d['transport_sweeps'])]}))" >> gpurun_out/r2f_banded_ab.jsonl
  done
done
echo "ab done"
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_async.py -q -x > gpurun_out/r2f_gputests.log 2>&1; echo "gpu tests rc=$?"
PHJ_CERT_LOG=gpurun_out/r2f_cert.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -k "c3 or c4 or c5_fp64" > gpurun_out/r2f_cert.log 2>&1; echo "cert rc=$?"
