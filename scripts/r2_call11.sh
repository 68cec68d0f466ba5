#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_bands.py -q > gpurun_out/r2k_bands_test.log 2>&1; echo "bands test rc=$?"
PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_timing.so timeout 600 python scripts/band_phases.py c5 > gpurun_out/r2k_band_phases.jsonl 2> gpurun_out/r2k_band_phases.err; echo "phases rc=$?"
timeout 600 python scripts/profile_step.py c5 float64 3 > gpurun_out/r2k_step.jsonl 2>&1; echo "step rc=$?"
