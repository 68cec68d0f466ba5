#!/bin/bash
timeout 900 python scripts/scaling_projection.py c5 float64 work > gpurun_out/r2s_scaling_work.json 2> gpurun_out/r2s_scaling.err; echo "work rc=$?"
timeout 900 python scripts/scaling_projection.py c5 float64 nodes > gpurun_out/r2s_scaling_nodes.json 2>> gpurun_out/r2s_scaling.err; echo "nodes rc=$?"
timeout 600 python bench.py > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; echo "bench rc=$?"
