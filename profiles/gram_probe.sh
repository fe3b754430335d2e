#!/bin/bash
# Build and run profiles/gram_probe.cu against the in-tree libatk_cuda.so.
set -e
cd "$(dirname "$0")/.."
nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_2010_10131_b200/csrc -I include \
  profiles/gram_probe.cu -o gpurun_out/gram_probe -L paper_2010_10131_b200 -l:libatk_cuda.so \
  -Xlinker -rpath -Xlinker "$PWD/paper_2010_10131_b200"
gpurun_out/gram_probe
