#!/bin/bash
mkdir -p gpurun_out
for sp in 0 1; do
  PHJ_COLOUR_SPLIT_SPATIAL=$sp timeout 1500 python scripts/scaling_projection.py c5 float64 work > gpurun_out/r2ao_scaling_projection_c5_spatial$sp.json 2>> gpurun_out/r2ao.err; echo "rc=$?"
done
python - <<'PY'
import json
for sp in (0,1):
    d=json.load(open(f'gpurun_out/r2ao_scaling_projection_c5_spatial{sp}.json'))
    for G in (2,4,8):
        g=d[f'G{G}']; print('spatial',sp,'G',G,'step',round(g['step_ms'],1),'eff',round(g['efficiency'],3),'tr',[round(x,1) for x in g['transport_ms_per_rank']])
PY
tail -2 gpurun_out/r2ao.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 scripts/multi_rank_check.py c5 129 2>&1 | grep -E "^rank|MULTI"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 scripts/multi_rank_check.py c3 65 2>&1 | grep -E "^rank|MULTI"
