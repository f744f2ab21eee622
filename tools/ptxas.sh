#!/bin/bash
# ptxas register/spill report for one CUDA source: tools/ptxas.sh sparse_fused.cu
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xptxas -v --expt-relaxed-constexpr -I include -I paper_2505_19586_b200/csrc -c "paper_2505_19586_b200/csrc/$1" \
  -o /tmp/ptxas_check.o 2>&1 | grep -E "error|spill|Used|Compiling entry" | sed 's/ptxas info    : //'
