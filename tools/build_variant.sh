#!/bin/bash
# build a variant of the library with extra nvcc flags:  tools/build_variant.sh NAME -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p tools/_variants/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include "$@" \
  -shared -o tools/_variants/$name/libtwilight.so paper_2502_02770_b200/csrc/*.cu -lcudart_static
