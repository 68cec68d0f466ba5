#!/bin/bash
# all-unreached tile early-out: kernel times, parity tests
mkdir -p gpurun_out
for c in c5 c3; do
  timeout 400 python scripts/band_ab.py $c >> gpurun_out/r2ah_skip_unreached_ab.jsonl 2>> gpurun_out/r2ah.err
done
cat gpurun_out/r2ah_skip_unreached_ab.jsonl | cut -c1-420; tail -3 gpurun_out/r2ah.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py tests/test_gpu_pruning.py -x -q > gpurun_out/r2ah_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2ah_tests.log
for spec in "c5 float64" "c5 float32" "c3 float64" "c4 float64" "c2 float64"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --dtype $2 --no-cpu-baseline --steps 5 >> gpurun_out/r2ah_bench.jsonl 2>> gpurun_out/r2ah.err
done
python -c "
import json
for l in open('gpurun_out/r2ah_bench.jsonl'):
    d=json.loads(l); print(d['config']['name'], d['dtype'], round(d['ms_per_step'],2), 'ms', round(d['roofline']['frac'],3), d['phases_ms'])
"
