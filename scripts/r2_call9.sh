#!/bin/bash
for cfg in "1 6,2 0" "1 6,2 1" "1 6,2 2" "2 3,1 0" "2 3,1 2" "2 4,1 2" "3 2,1 2" "1 4,1 2" "2 2,1 3"; do
  set -- $cfg
  PHJ_BAND_SCALE=$1 PHJ_SOLVE_BAND_WINDOW=$2 PHJ_BAND_INNER=$3 timeout 300 python scripts/band_ab.py c5 >> gpurun_out/r2i_band_ab.jsonl 2>> gpurun_out/r2i_band_ab.err
done
echo done
