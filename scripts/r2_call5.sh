#!/bin/bash
# C5 fp64: phase split, ncu captures of the two dominant kernels, sanitizers on reduced runs
PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_timing.so timeout 600 python scripts/phase_cycles.py c5 float64 > gpurun_out/r2e_c5_phase_cycles.json 2> gpurun_out/r2e_phase.err; echo "phase rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_async_kernel -c 1 -o gpurun_out/r2e_c5_solve_async python scripts/profile_step.py c5 float64 1 > gpurun_out/r2e_ncu_solve.log 2>&1; echo "ncu solve rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"transport_kernel<" -c 1 -o gpurun_out/r2e_c5_transport python scripts/profile_step.py c5 float64 1 > gpurun_out/r2e_ncu_transport.log 2>&1; echo "ncu transport rc=$?"
timeout 900 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_run.py > gpurun_out/r2e_memcheck.log 2>&1; echo "memcheck rc=$?"
