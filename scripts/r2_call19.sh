#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/step_breakdown.py c5 float64 > gpurun_out/r2s_step_breakdown.jsonl 2> gpurun_out/r2s_step_breakdown.err; echo "breakdown rc=$?"
cat gpurun_out/r2s_step_breakdown.jsonl
timeout 600 python scripts/profile_step.py c5 float64 1 > gpurun_out/r2s_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_c5f64_launches.csv python scripts/profile_step.py c5 float64 1 > gpurun_out/r2s_ncu_list.log 2>&1; echo "launches rc=$?"
