python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in head cur; do
  for c in "C2" "C4 --batch 16" "C3"; do
    TW_LIB_PATH=tools/_variants/$v/libtwilight.so timeout 300 python tools/stage_time.py --config $c --layers 1 2>&1 | tail -1
  done
  TW_LIB_PATH=tools/_variants/$v/libtwilight.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', 'bench', d['value'], d['dense_us_per_layer'], d['e2e']['value'])"
done
