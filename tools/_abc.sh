#!/bin/bash
# bench lines of library variants x attention chunk sizes:  tools/_abc.sh "C2 C5" "0 256 128" VARIANT...
cd "$(dirname "$0")/.."
cfgs=$1; chunks=$2; shift 2
for r in 1 2; do
for c in $cfgs; do
for ch in $chunks; do
for v in "$@"; do
  TW_LIB_PATH=tools/_variants/$v/libtwilight.so timeout 300 python bench.py --config $c --chunk $ch --no-cpu-baseline 2>/dev/null \
    | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_us']; print('$c', 'chunk $ch', '$v', d['value'], 'dense', d['dense_us_per_layer'], 'K4', k['K4_attention'], 'attn', k.get('K4a_attn_kernel'))"
done; done; done; done
