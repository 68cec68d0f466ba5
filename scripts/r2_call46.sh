#!/bin/bash
mkdir -p gpurun_out
for pf in 0 1; do
  PHJ_PHI_PREFILL=$pf timeout 600 python bench.py --no-cpu-baseline --steps 8 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('prefill $pf', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), d['phases_ms'])"
done
PHJ_PHI_PREFILL=1 timeout 600 python bench.py --no-cpu-baseline --steps 5 --config c3 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('c3 prefill 1', round(d['ms_per_step'],2), d['phases_ms'])"
PHJ_PHI_PREFILL=0 timeout 600 python bench.py --no-cpu-baseline --steps 5 --config c3 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('c3 prefill 0', round(d['ms_per_step'],2), d['phases_ms'])"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py tests/test_gpu_api.py -x -q 2>&1 | tail -3
