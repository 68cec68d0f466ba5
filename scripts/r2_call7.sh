#!/bin/bash
# banded patch solve + capped transport bands: speed A/B and correctness
for c in c5 c3 c4 c2; do
  for sb in 0 1; do
    PHJ_SOLVE_BANDED=$sb timeout 600 python scripts/profile_step.py $c float64 3 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'config':d['config'],'solve_banded':$sb,'patch_kernel_ms':d['patch_kernel']['kernel_ms'],'executed':d['patch_kernel'].get('performed'),'transport_ms':d['transport_kernel']['kernel_ms'],'phases':d['phases_ms'],'psweeps':[min(d['patch_sweeps']),max(d['patch_sweeps'])],'tsweeps':[min(d['transport_sweeps']),max(d['transport_sweeps'])]}))" >> gpurun_out/r2g_banded_solve_ab.jsonl
  done
done
echo "ab done"
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_api.py -q -x > gpurun_out/r2g_gputests.log 2>&1; echo "gpu tests rc=$?"
PHJ_CERT_LOG=gpurun_out/r2g_cert.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -k "c2_fp64 or c3 or c4 or c5_fp64" > gpurun_out/r2g_cert.log 2>&1; echo "cert rc=$?"
