#!/bin/bash
# ncu capture of the banded patch-solve pass at C5 fp64 (after a clean plain run); raw + source pages
mkdir -p gpurun_out
timeout 600 python scripts/profile_step.py c5 float64 1 > gpurun_out/r2aa_plain.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:^solve_kernel$ --launch-skip 1 -c 1 -o gpurun_out/r2aa_c5_solve python scripts/profile_step.py c5 float64 1 > gpurun_out/r2aa_ncu_solve.log 2>&1; echo "ncu solve rc=$?"
ncu -i gpurun_out/r2aa_c5_solve.ncu-rep --page source --csv --print-source sass > gpurun_out/r2aa_c5_solve_sass.csv 2>/dev/null; echo "export rc=$?"
ncu -i gpurun_out/r2aa_c5_solve.ncu-rep --page raw --csv > gpurun_out/r2aa_c5_solve_raw.csv 2>/dev/null
ls -la gpurun_out | grep r2aa
