#!/bin/bash
timeout 900 python scripts/transport_act_ab.py > gpurun_out/r2q_act_ab.jsonl 2> gpurun_out/r2q_act_ab.err; echo "act rc=$?"
