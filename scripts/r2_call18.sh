#!/bin/bash
# A/B of the barrier-free value-ordered patch-solve pass (PHJ_BAND_ASYNC 0/1), then certificates and bench with it on
mkdir -p gpurun_out
for ba in 0 1; do
  for c in c5 c3; do
    PHJ_BAND_ASYNC=$ba timeout 400 python scripts/band_ab.py $c | sed "s/^{/{\"band_async\": $ba, /" >> gpurun_out/r2r_band_async_ab.jsonl 2>> gpurun_out/r2r_band_async_ab.err
  done
done
cat gpurun_out/r2r_band_async_ab.jsonl
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c5_fp64" > gpurun_out/r2r_cert_band_async.log 2>&1; echo "cert rc=$?"
tail -5 gpurun_out/r2r_cert_band_async.log
timeout 600 python bench.py > gpurun_out/r2r_bench_c5f64.json 2> gpurun_out/r2r_bench.err; echo "bench rc=$?"
cat gpurun_out/r2r_bench_c5f64.json
