#!/bin/bash
mkdir -p gpurun_out
export PHJ_AB_TRANSPORT_ONLY=1
for v in tch1 default tch4; do
  L=""; [ "$v" != default ] && L=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so
  for c in c5 c3; do PHJ_LIB_PATH=$L timeout 400 python scripts/band_ab.py $c 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', d['config'], 'G1', round(d['G1_transport_ms'],1), 'G8', round(d['G8_transport_ms'],1), d['G1_tsweeps'])"; done
done
unset PHJ_AB_TRANSPORT_ONLY
timeout 900 python scripts/transport_sweep_floor.py c5 2>/dev/null | tail -6
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
