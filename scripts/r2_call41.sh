#!/bin/bash
# two ranks on one GPU (gloo) through the whole pipeline incl. the sharded feedback; transport occupancy variants
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_async.py -x -q -k "sharded or slabs" 2>&1 | tail -2
for spec in "c5 129" "c3 65" "c2 257" "c4 41"; do
  set -- $spec
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 scripts/multi_rank_check.py $1 $2 2>&1 | grep -E "rank|MULTI" >> gpurun_out/r2am_multi_rank_check.txt
done
cat gpurun_out/r2am_multi_rank_check.txt
export PHJ_AB_TRANSPORT_ONLY=1
for v in t3 t4; do
  PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so timeout 400 python scripts/band_ab.py c5 >> gpurun_out/r2am_transport_occupancy.jsonl 2>> gpurun_out/r2am.err
done
timeout 400 python scripts/band_ab.py c5 >> gpurun_out/r2am_transport_occupancy.jsonl 2>> gpurun_out/r2am.err
cut -c1-330 gpurun_out/r2am_transport_occupancy.jsonl; tail -2 gpurun_out/r2am.err
