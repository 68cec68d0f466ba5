#!/bin/bash
# ncu source-level capture of the banded 3D transport kernel at C5 fp64 (after a clean plain run)
mkdir -p gpurun_out
timeout 600 python scripts/profile_step.py c5 float64 1 > gpurun_out/r2w_plain.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:^transport_kernel$ -c 1 -o gpurun_out/r2w_c5_transport python scripts/profile_step.py c5 float64 1 > gpurun_out/r2w_ncu_transport.log 2>&1; echo "ncu transport rc=$?"
ls -la gpurun_out/
ncu -i gpurun_out/r2w_c5_transport.ncu-rep --page source --csv --print-source sass > gpurun_out/r2w_c5_transport_sass.csv 2>/dev/null; echo "export rc=$?"
ncu -i gpurun_out/r2w_c5_transport.ncu-rep --page raw --csv > gpurun_out/r2w_c5_transport_raw.csv 2>/dev/null
