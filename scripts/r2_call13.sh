#!/bin/bash
timeout 600 python scripts/debug_spurious.py 257 > gpurun_out/r2m_spurious.log 2>&1; echo "dbg rc=$?"
for v in wpipe both; do
  PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so timeout 300 python scripts/band_ab.py c5 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/r2m_variant_ab.jsonl 2>> gpurun_out/r2m_variant_ab.err
done
