#!/bin/bash
# tools/variant.sh NAME [extra nvcc flags...] -> build/variants/NAME.so (+ ptxas spill report)
set -e -o pipefail
name=$1; shift
mkdir -p build/variants
log=$(mktemp)
if ! nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -prec-div=false -prec-sqrt=false -ftz=true -Xptxas -v "$@" \
  -o build/variants/$name.so paper_2603_00280_b200/csrc/mf_kernels.cu -ldl > "$log" 2>&1; then
  grep -i "error" "$log" | head -20; rm -f "$log"; exit 1
fi
grep -A2 "path_kernel\|pool_kernel" "$log" | grep -o "Compiling entry.*\|[0-9]* bytes stack frame, [0-9]* bytes spill stores, [0-9]* bytes spill loads" | paste - - | sed -E 's/Compiling entry function .*(path|pool)_kernelI(L[ib][0-9]*E)?(L[ib][0-9]*E)?.*for .sm_100a.\s*/\1 \2\3 /' || true
rm -f "$log"
