#!/bin/bash
# slab feedback test, multi-GPU projection, ncu captures of the two dominant kernels in their final form
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_async.py -x -q -k slabs > gpurun_out/r2ae_slab_test.log 2>&1; echo "slab test rc=$?"; tail -3 gpurun_out/r2ae_slab_test.log
timeout 1200 python scripts/scaling_projection.py c5 float64 work > gpurun_out/r2ae_scaling_projection_c5.json 2> gpurun_out/r2ae_scaling.err; echo "projection rc=$?"
timeout 1200 python scripts/scaling_projection.py c5 float64 nodes > gpurun_out/r2ae_scaling_projection_c5_nodelpt.json 2>> gpurun_out/r2ae_scaling.err; echo "projection(nodes) rc=$?"
timeout 600 python scripts/profile_step.py c5 float64 1 > gpurun_out/r2ae_plain.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:^solve_kernel$ --launch-skip 1 -c 1 -o gpurun_out/r2ae_c5_solve python scripts/profile_step.py c5 float64 1 > gpurun_out/r2ae_ncu_solve.log 2>&1; echo "ncu solve rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:^transport_kernel$ -c 1 -o gpurun_out/r2ae_c5_transport python scripts/profile_step.py c5 float64 1 > gpurun_out/r2ae_ncu_transport.log 2>&1; echo "ncu transport rc=$?"
ncu -i gpurun_out/r2ae_c5_solve.ncu-rep --page source --csv --print-source sass > gpurun_out/r2ae_c5_solve_sass.csv 2>/dev/null
ncu -i gpurun_out/r2ae_c5_transport.ncu-rep --page source --csv --print-source sass > gpurun_out/r2ae_c5_transport_sass.csv 2>/dev/null
ls -la gpurun_out | grep r2ae
