#!/bin/bash
for v in nb4 nb4c1; do
  PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so timeout 300 python scripts/band_ab.py c5 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/r2p_variant_ab.jsonl 2>> gpurun_out/r2p_variant_ab.err
  PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so PHJ_CERT_N=129 timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -k "c3 or c5_fp64" > gpurun_out/r2p_cert_$v.log 2>&1; echo "$v cert rc=$?"
done
