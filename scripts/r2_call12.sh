#!/bin/bash
for v in default wpipe minint both; do
  if [ $v = default ]; then L=$PWD/paper_1109_3577_b200/_lib/libphj.so; else L=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so; fi
  PHJ_LIB_PATH=$L timeout 300 python scripts/band_ab.py c5 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/r2l_variant_ab.jsonl 2>> gpurun_out/r2l_variant_ab.err
done
echo "ab done"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2l_gputests.log 2>&1; echo "gpu tests rc=$?"
