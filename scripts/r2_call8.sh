#!/bin/bash
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --config c5 --dtype float32 --no-cpu-baseline > gpurun_out/r2h_bench_c5f32.json 2>> gpurun_out/r2h_bench.err; echo "bench f32 rc=$?"
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r2h_bench_c3.json 2>> gpurun_out/r2h_bench.err; echo "bench c3 rc=$?"
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2h_bench_c2.json 2>> gpurun_out/r2h_bench.err; echo "bench c2 rc=$?"
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2h_bench_c4.json 2>> gpurun_out/r2h_bench.err; echo "bench c4 rc=$?"
timeout 900 python scripts/scaling_projection.py c5 float64 > gpurun_out/r2h_scaling_c5.json 2> gpurun_out/r2h_scaling.err; echo "scaling rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_c5f64_launches.csv python scripts/profile_step.py c5 float64 1 > gpurun_out/r2h_ncu_list.log 2>&1; echo "launches rc=$?"
