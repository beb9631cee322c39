for v in T256G2:"-DTW_SEL_THREADS=256 -DTW_SEL_GROUPS=2" T128G1:"-DTW_SEL_THREADS=128 -DTW_SEL_GROUPS=1" T256G1:"-DTW_SEL_THREADS=256 -DTW_SEL_GROUPS=1"; do
  name=${v%%:*}; flags=${v#*:}; bash tools/build_variant.sh $name $flags > /dev/null 2>&1 &
done
wait
timeout 900 python -m pytest tests/test_gpu_api.py -x -q 2>&1 | tail -2
for c in C2 C5; do
  echo -n "base "; timeout 300 python tools/stage_time.py --config $c --layers 1 2>&1 | tail -1 | grep -o '"K2_select": [0-9.]*'
  for name in T256G2 T128G1 T256G1; do echo -n "$name "; TW_LIB_PATH=tools/_variants/$name/libtwilight.so timeout 300 python tools/stage_time.py --config $c --layers 1 2>&1 | tail -1 | grep -o '"K2_select": [0-9.]*'; done
done
TW_LIB_PATH=tools/_variants/T128G1/libtwilight.so timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
