#!/bin/bash
# transport: occupancy variants (CTAs/SM x colours per batch) and band width
mkdir -p gpurun_out
export PHJ_AB_TRANSPORT_ONLY=1
for v in t2c1 t3c1 t4c1; do
  for c in c5 c3; do
    PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so timeout 400 python scripts/band_ab.py $c >> gpurun_out/r2y_transport_variants.jsonl 2>> gpurun_out/r2y_transport_variants.err
  done
done
for ts in 1 1.5 2 3; do
  for tw in "3,1" "2,1" "4,2"; do
    PHJ_TBAND_SCALE=$ts PHJ_TRANSPORT_BAND_WINDOW=$tw timeout 400 python scripts/band_ab.py c5 >> gpurun_out/r2y_transport_variants.jsonl 2>> gpurun_out/r2y_transport_variants.err
  done
done
cat gpurun_out/r2y_transport_variants.jsonl; tail -3 gpurun_out/r2y_transport_variants.err
