#!/bin/bash
# A/B of the conical pre-pass (PHJ_BAND_CONE = r: controls within pi/r of the lifted feedback in the value-ordered pass)
mkdir -p gpurun_out
for r in 0 4 3 6 8; do
  for c in c5 c3; do
    PHJ_BAND_CONE=$r timeout 400 python scripts/band_ab.py $c >> gpurun_out/r2t_cone_ab.jsonl 2>> gpurun_out/r2t_cone_ab.err
  done
done
cat gpurun_out/r2t_cone_ab.jsonl
tail -5 gpurun_out/r2t_cone_ab.err
