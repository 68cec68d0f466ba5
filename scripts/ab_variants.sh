#!/bin/bash
# Time the workload pipeline with each built kernel variant: ab_variants.sh <config> <dtype> names...
cd "$(dirname "$0")/.."
cfg=$1; dt=$2; shift 2
for v in "$@"; do
  echo "== $v"
  PHJ_LIB_PATH=$PWD/paper_1109_3577_b200/_lib/variants/libphj_$v.so python -u scripts/profile_step.py $cfg $dt 2 | tail -1
done
