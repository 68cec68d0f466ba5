#!/bin/bash
# Build kernel variants for A/B timing (scripts/ab_variants.sh); outputs are git-ignored .so files.
set -e
cd "$(dirname "$0")/.."
OUT=paper_1109_3577_b200/_lib/variants
mkdir -p $OUT
build() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr "$@" -o $OUT/libphj_$name.so \
    paper_1109_3577_b200/csrc/phj_solve.cu paper_1109_3577_b200/csrc/phj_ops.cu paper_1109_3577_b200/csrc/phj_bands.cu &
}
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  build $name $flags
done
wait
ls $OUT
