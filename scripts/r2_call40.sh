#!/bin/bash
# final validation: smoke, full GPU suite, default bench + reference arm, other configs
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2al_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2al_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2al_gputests_full_suite.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2al_gputests_full_suite.log
timeout 900 python bench.py > gpurun_out/r2al_bench_c5f64.json 2> gpurun_out/r2al_bench.err; echo "bench rc=$?"
cat gpurun_out/r2al_bench_c5f64.json | cut -c1-1500
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2al_bench_reference_c5.json 2>> gpurun_out/r2al_bench.err; echo "ref rc=$?"
for spec in "c5 float32" "c3 float64" "c4 float64" "c2 float64" "c2 float32" "c1 float64"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --dtype $2 --no-cpu-baseline >> gpurun_out/r2al_bench_other_configs.jsonl 2>> gpurun_out/r2al_bench.err
done
python -c "
import json
for l in open('gpurun_out/r2al_bench_other_configs.jsonl'):
    d=json.loads(l); print(d['config']['name'], d['dtype'], round(d['ms_per_step'],2), 'ms', 'e2e', round(d['e2e']['ms_per_step'],2), round(d['roofline']['frac'],3))
"
tail -3 gpurun_out/r2al_bench.err
