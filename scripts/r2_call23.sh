#!/bin/bash
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2w_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2w_bench_ref.json 2> gpurun_out/r2w_bench_ref.err; echo "ref rc=$?"
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2w_gputests.log 2>&1; echo "gpu tests rc=$?"
