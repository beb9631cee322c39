timeout 600 python -m pytest tests/test_gpu_topp.py tests/test_gpu_decode.py -x -q 2>&1 | tail -3
bash tools/trace_topp.sh
for c in C2 C5; do TW_LIB_PATH=/tmp/twtrace/libtwilight.so timeout 300 python tools/topp_trace.py --config $c 2>&1 | tail -14; done
for c in C2 C5 C3; do timeout 300 python tools/stage_time.py --config $c --layers 1 2>&1 | tail -1; done
