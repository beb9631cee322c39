bash tools/trace_topp.sh
for c in C2 C5; do TW_LIB_PATH=/tmp/twtrace/libtwilight.so timeout 300 python tools/prof_step.py --config $c --reps 1 2>&1 | tail -8; done
