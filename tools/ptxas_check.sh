#!/bin/bash
# registers / spills of the kernels of one source file: tools/ptxas_check.sh pde.cu [regex]
cd "$(dirname "$0")/../paper_2109_04131_b200/csrc" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xptxas -v -c "$1" -o /tmp/ptxas_check.o 2>&1 \
  | grep -A3 "${2:-Compiling entry}" | grep "error\|entry\|spill\|Used" | sed 's/ptxas info    : //'
