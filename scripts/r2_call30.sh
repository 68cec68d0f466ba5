#!/bin/bash
# full GPU suite, default bench (C5 fp64) + reference arm, other configs, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2ad_gputests_full_suite.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2ad_gputests_full_suite.log
timeout 900 python bench.py > gpurun_out/r2ad_bench_c5f64.json 2> gpurun_out/r2ad_bench.err; echo "bench rc=$?"
cat gpurun_out/r2ad_bench_c5f64.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2ad_bench_reference_c5.json 2>> gpurun_out/r2ad_bench.err; echo "ref rc=$?"
for spec in "c5 float32" "c3 float64" "c4 float64" "c2 float64" "c2 float32" "c1 float64"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --dtype $2 --no-cpu-baseline >> gpurun_out/r2ad_bench_other_configs.jsonl 2>> gpurun_out/r2ad_bench.err
done
python -c "
import json
for l in open('gpurun_out/r2ad_bench_other_configs.jsonl'):
    d=json.loads(l); print(d['config']['name'], d['dtype'], round(d['ms_per_step'],2), 'ms', d['roofline']['frac'])
"
timeout 600 python scripts/profile_step.py c5 float64 1 > gpurun_out/r2ad_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ad_c5f64_launches.csv python scripts/profile_step.py c5 float64 1 > gpurun_out/r2ad_ncu_list.log 2>&1; echo "launches rc=$?"
