#!/bin/bash
mkdir -p gpurun_out
PHJ_AB_TRANSPORT_ONLY=1 timeout 400 python scripts/band_ab.py c5 2>/dev/null | cut -c1-330
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
timeout 1500 python scripts/scaling_projection.py c5 float64 work > gpurun_out/r2ar_scaling_projection_c5.json 2> gpurun_out/r2ar.err; echo "projection rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2ar_scaling_projection_c5.json'))
for G in (1,2,4,8):
    g=d[f'G{G}']; print('G',G,'step',round(g['step_ms'],1),'eff',round(g['efficiency'],3),'tr',[round(x,1) for x in g['transport_ms_per_rank']],'pa max',round(max(g['patch_ms_per_rank']),1))
PY
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 scripts/multi_rank_check.py c5 129 2>&1 | grep -E "^rank|MULTI"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 scripts/multi_rank_check.py c4 41 2>&1 | grep -E "^rank|MULTI"
