#!/bin/bash
# build a traced copy of the library (per-CTA phase timestamps of the top-p kernels)
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/twtrace
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I include -DTW_TOPP_TRACE \
  -shared -o /tmp/twtrace/libtwilight.so paper_2502_02770_b200/csrc/*.cu -lcudart_static
