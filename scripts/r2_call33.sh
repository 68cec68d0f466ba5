#!/bin/bash
# activity filter of the value-ordered pass: A/B, parity tests, certificates
mkdir -p gpurun_out
for f in 0 1; do
  for c in c5 c3; do
    PHJ_BAND_FILTER=$f timeout 400 python scripts/band_ab.py $c | sed "s/^{/{\"band_filter\": $f, /" >> gpurun_out/r2ag_band_filter_ab.jsonl 2>> gpurun_out/r2ag_band_filter_ab.err
  done
done
cat gpurun_out/r2ag_band_filter_ab.jsonl | cut -c1-420; tail -3 gpurun_out/r2ag_band_filter_ab.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py tests/test_gpu_pruning.py -x -q > gpurun_out/r2ag_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2ag_tests.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c5" > gpurun_out/r2ag_cert.log 2>&1; echo "cert rc=$?"; tail -4 gpurun_out/r2ag_cert.log
