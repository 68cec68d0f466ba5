#!/bin/bash
# round 2 first look: C5 fp64 step profile, bench line, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python scripts/profile_step.py c5 float64 3 > gpurun_out/r2a_c5f64_step.jsonl 2> gpurun_out/r2a_c5f64_step.err
python bench.py --config c5 --dtype float64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_c5f64.json 2> gpurun_out/r2a_bench_c5f64.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2a_c5f64_launches.csv python scripts/profile_step.py c5 float64 1 > gpurun_out/r2a_ncu.log 2>&1
tail -3 gpurun_out/*.err
