#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/colour_activity.py c5 > gpurun_out/r2v_colour_activity.json 2> gpurun_out/r2v_colour_activity.err; echo "rc=$?"
cat gpurun_out/r2v_colour_activity.json; tail -3 gpurun_out/r2v_colour_activity.err
