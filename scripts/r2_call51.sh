#!/bin/bash
mkdir -p gpurun_out
timeout 900 python scripts/transport_sweep_floor.py c5 2>/dev/null | tail -6
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
export PHJ_AB_TRANSPORT_ONLY=1
for c in c5 c3 c4; do timeout 400 python scripts/band_ab.py $c 2>/dev/null | cut -c1-330; done
