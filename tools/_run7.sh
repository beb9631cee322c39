set -e
for v in base:"" nocand:"-DTW_X_NOCAND" noj:"-DTW_X_NOJ" both:"-DTW_X_NOCAND -DTW_X_NOJ"; do
  name=${v%%:*}; flags=${v#*:}
  mkdir -p /tmp/tw_$name
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I include -DTW_TOPP_TRACE $flags -shared -o /tmp/tw_$name/libtwilight.so paper_2502_02770_b200/csrc/*.cu -lcudart_static &
done
wait
for name in base nocand noj both; do echo "== $name"; TW_LIB_PATH=/tmp/tw_$name/libtwilight.so timeout 300 python tools/topp_trace.py --config C2 2>&1 | grep -A1 resolve | tail -2; done
