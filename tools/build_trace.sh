#!/bin/sh
# Build a trace / microbenchmark tool from tools/<name>.cu against the in-tree library:
#   sh tools/build_trace.sh attn_bwd_trace   ->  tools/attn_bwd_trace_bin
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2505_11580_b200/csrc \
    "tools/$1.cu" -o "tools/$1_bin" -L paper_2505_11580_b200 -lfipa_b200 -Xlinker -rpath='$ORIGIN/../paper_2505_11580_b200' -lcuda
