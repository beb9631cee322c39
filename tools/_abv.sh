#!/bin/bash
# bench lines of several library variants:  tools/_abv.sh "C2 C5" VARIANT...
cd "$(dirname "$0")/.."
cfgs=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
for c in $cfgs; do
for v in "$@"; do
  TW_LIB_PATH=tools/_variants/$v/libtwilight.so timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/abv_${v}_${c}.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/abv_${v}_${c}.json').read().strip().splitlines()[-1]);print('$c','$v',d['value'],'dense',d.get('dense_us_per_layer'),d.get('kernels_us'))" 2>&1 | tail -1
done; done; done
