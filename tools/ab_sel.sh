set -u
mkdir -p gpurun_out
TW_SEL_THREADS=1024 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/sel_test.log 2>&1; echo "tests(1024): $(tail -1 gpurun_out/sel_test.log)"
run() {  # tag env... config
  local tag=$1 c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/ab_${tag}_${c}.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${tag}_${c}.json').read().strip().splitlines()[-1]);print('$c','$tag',d['ms_per_step'],d.get('kernels_us'))"
}
for c in C2 C5 C4 C1; do
  run base $c X=1
  run t1024 $c TW_SEL_THREADS=1024
  run st4 $c TW_LIB_PATH=tools/_variants/st4/libtwilight.so
done
