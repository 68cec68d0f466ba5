#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python scripts/scaling_projection.py c5 float64 work > gpurun_out/r2aj_scaling_projection_c5.json 2> gpurun_out/r2aj_scaling.err; echo "projection rc=$?"
timeout 1500 python scripts/scaling_projection.py c5 float64 nodes > gpurun_out/r2aj_scaling_projection_c5_nodelpt.json 2>> gpurun_out/r2aj_scaling.err; echo "projection(nodes) rc=$?"
tail -3 gpurun_out/r2aj_scaling.err
