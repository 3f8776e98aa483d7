#!/bin/bash
# builds chol5_<NT> for NT in $@ (default 256 512)
cd "$(dirname "$0")"
for t in ${@:-256 512}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -DNTH=$t -I../../paper_2602_17601_b200/csrc chol5.cu -o chol5_$t 2>&1 | grep -E "error|registers|spill"
done
