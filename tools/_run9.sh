bash tools/build_variant.sh Q2 -DTW_QM_STAGES=2 > /dev/null 2>&1
for c in C2 C5; do
  echo -n "base "; timeout 300 python tools/stage_time.py --config $c --layers 1 2>&1 | tail -1 | grep -o '"K2_select": [0-9.]*'
  echo -n "Q2 "; TW_LIB_PATH=tools/_variants/Q2/libtwilight.so timeout 300 python tools/stage_time.py --config $c --layers 1 2>&1 | tail -1 | grep -o '"K2_select": [0-9.]*'
done
