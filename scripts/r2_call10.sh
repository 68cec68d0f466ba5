#!/bin/bash
for cfg in "6,2 3,1" "5,2 2,1" "8,2 4,1" "6,1 3,0" "4,2 2,0" "7,3 3,2"; do
  set -- $cfg
  PHJ_SOLVE_BAND_WINDOW=$1 PHJ_TRANSPORT_BAND_WINDOW=$2 timeout 300 python scripts/band_ab.py c5 >> gpurun_out/r2j_band_ab.jsonl 2>> gpurun_out/r2j_band_ab.err
done
echo done
