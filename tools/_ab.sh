python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in lean_m2 lean2_m2; do
  for c in "C2" "C4 --batch 16" "C3"; do
    TW_LIB_PATH=tools/_variants/$v/libtwilight.so timeout 300 python tools/stage_time.py --config $c --layers 1 2>&1 | tail -1
  done
done
