#!/bin/bash
# One profiling pass for profiles/ (run on the GPU box):  tools/profile_round.sh <tag>
#   GPU tests; bench lines C1-C5 (ours) and the reference arm; the launch list of
#   the C2 bench command (ncu gpu__time_duration, cold/serialised); one ncu
#   --set full capture of each config's step kernels (summary + per-stage DRAM
#   traffic -> ncu_traffic.json); the opt-in fused per-unit kernel (TW_UNIT=1)
#   bench line and phase trace (needs tools/_variants/utrace, built with
#   tools/build_variant.sh utrace -DTW_UNIT_TRACE -DTW_TOPP_TRACE).
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_${TAG}.log 2>&1; tail -2 gpurun_out/gputest_${TAG}.log
for c in C2 C1 C3 C5 C4; do
  timeout 900 python bench.py --config $c $([ $c != C2 ] && echo --no-cpu-baseline) > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  tail -c 300 gpurun_out/bench_${TAG}_$c.json
done
for c in C2 C1 C3 C5; do
  timeout 900 python bench.py --impl reference --config $c > gpurun_out/bench_ref_${TAG}_$c.json 2>&1
done
TW_UNIT=1 timeout 900 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_${TAG}_C2_unit.json 2>&1
for c in C2 C5 C3; do
  TW_UNIT=1 TW_LIB_PATH=tools/_variants/utrace/libtwilight.so timeout 300 python tools/unit_trace.py --config $c \
    --json gpurun_out/unit_trace_${TAG}_$c.json > /dev/null 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_${TAG}_C2.csv --json gpurun_out/launches_${TAG}_C2.json | grep "tw::" || true
for c in C1 C2 C3 C5 C4; do
  timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"attn_kernel|quest_select|topp_unit|topp_head|estimate_kernel|quest_filter|append_kernel|merge_kernel|unit_step" -c 8 \
    -o /tmp/full_${TAG}_$c python tools/prof_step.py --config $c --reps 1 > /dev/null 2>&1
  # reports stay on the box (gpurun_out/ merges back only up to 64 MiB): summaries + traffic come back
  python tools/ncu_hot.py /tmp/full_${TAG}_$c.ncu-rep . --lines 6 > gpurun_out/ncu_full_${TAG}_$c.txt 2>&1
  python tools/traffic_json.py /tmp/full_${TAG}_$c.ncu-rep $c > gpurun_out/traffic_${TAG}_$c.json 2>&1 || true
done
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
