#!/bin/bash
# tools/variant.sh NAME [extra nvcc flags...] -> build/variants/NAME.so (+ ptxas spill report)
set -e
name=$1; shift
mkdir -p build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -prec-div=false -prec-sqrt=false -ftz=true -Xptxas -v "$@" \
  -o build/variants/$name.so paper_2603_00280_b200/csrc/mf_kernels.cu 2>&1 \
  | grep -A2 "path_kernel" | grep -o "Compiling entry.*\|[0-9]* bytes stack frame, [0-9]* bytes spill stores, [0-9]* bytes spill loads" | paste - - | sed -E 's/Compiling entry function .*path_kernelILi([0-9])ELb([01]).*for .sm_100a.\s*/k<\1,\2> /'
