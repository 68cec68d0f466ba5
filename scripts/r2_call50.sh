#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2aq_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2aq_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2aq_gputests_full_suite.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2aq_gputests_full_suite.log
timeout 900 python bench.py > gpurun_out/r2aq_bench_c5f64.json 2> gpurun_out/r2aq_bench.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/r2aq_bench_c5f64.json
