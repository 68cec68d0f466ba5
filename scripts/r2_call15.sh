#!/bin/bash
# ncu captures of the round-2 dominant kernels at C5 fp64 (after a clean run)
timeout 300 python scripts/profile_step.py c5 float64 1 > gpurun_out/r2o_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:solve_kernel --launch-skip 1 -c 1 -o gpurun_out/r2o_c5_solve_banded python scripts/profile_step.py c5 float64 1 > gpurun_out/r2o_ncu_solve.log 2>&1; echo "ncu solve rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:transport_kernel -c 1 -o gpurun_out/r2o_c5_transport python scripts/profile_step.py c5 float64 1 > gpurun_out/r2o_ncu_transport.log 2>&1; echo "ncu transport rc=$?"
