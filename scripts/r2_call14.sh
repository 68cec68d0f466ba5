#!/bin/bash
for v in ctas3 u4 w4c4; do
  PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so timeout 300 python scripts/band_ab.py c5 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/r2n_variant_ab.jsonl 2>> gpurun_out/r2n_variant_ab.err
done
echo "ab done"
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2n_gputests.log 2>&1; echo "gpu tests rc=$?"
