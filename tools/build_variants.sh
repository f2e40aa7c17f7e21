#!/bin/bash
# Build library variants with extra -D flags into /root/repo/variants/<name>.so
# usage: tools/build_variants.sh name1 "-DFOO=1" name2 "-DBAR" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
FLAGS=$(python -c "from paper_2603_00280_b200 import build as b; print(' '.join(b.NVCC_FLAGS))" | sed 's/-Xptxas -v//')
pids=()
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  nvcc $FLAGS $defs -o variants/$name.so paper_2603_00280_b200/csrc/mf_kernels.cu -ldl &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
ls -la variants/
