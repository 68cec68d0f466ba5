#!/bin/bash
# round 2: GPU suite after the counter changes, quick certificates, default bench
nproc; free -g | head -2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gputests.log 2>&1; echo "gpu tests rc=$?"
PHJ_CERT_N=129 PHJ_CERT_LOG=gpurun_out/r2b_cert_small.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/r2b_cert_small.log 2>&1; echo "cert small rc=$?"
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2b_gputests.log gpurun_out/r2b_cert_small.log
