set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/est_test.log 2>&1; echo "tests: $(tail -1 gpurun_out/est_test.log)"
for v in "" st3 st6 st8; do for c in C2 C5 C1 C3; do
  lib=""; [ -n "$v" ] && lib=tools/_variants/$v/libtwilight.so
  TW_LIB_PATH=$lib timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/est_${c}_${v}.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/est_${c}_${v}.json').read().strip().splitlines()[-1]);print('$c','v=$v',d['ms_per_step'],d.get('kernels_us'))"
done; done
