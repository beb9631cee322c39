#!/bin/bash
# build the library as of git revision REV into tools/_variants/NAME:  tools/build_rev.sh NAME REV [nvcc flags]
set -e
cd "$(dirname "$0")/.."
name=$1; rev=$2; shift 2
tmp=$(mktemp -d)
git archive "$rev" paper_2502_02770_b200/csrc include | tar -x -C "$tmp"
mkdir -p tools/_variants/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I "$tmp/include" "$@" \
  -shared -o tools/_variants/$name/libtwilight.so "$tmp"/paper_2502_02770_b200/csrc/*.cu -lcudart_static
rm -rf "$tmp"
