#!/bin/bash
# stage times of several library variants:  tools/_abn.sh CONFIG VARIANT...
cd "$(dirname "$0")/.."
cfg=$1; shift
for r in 1 2; do
for v in "$@"; do
  echo -n "$v "; TW_LIB_PATH=tools/_variants/$v/libtwilight.so timeout 300 python tools/stage_time.py --config $cfg --layers 2 2>&1 | tail -1
done
done
