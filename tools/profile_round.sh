#!/bin/bash
# One profiling pass for profiles/ (run on the GPU box):  tools/profile_round.sh <tag>
#   bench lines (ours, reference arm, other configs), the launch list of the bench
#   command (ncu gpu__time_duration, cold/serialised), one ncu --set full capture of
#   the step's kernels (summary + per-stage DRAM traffic), GPU tests.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_${TAG}_C2.json 2> gpurun_out/bench_${TAG}_C2.err; tail -c 400 gpurun_out/bench_${TAG}_C2.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}_C2.json 2>&1; tail -c 300 gpurun_out/bench_ref_${TAG}_C2.json
for c in C1 C3 C5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_${TAG}_C2.csv --json gpurun_out/launches_${TAG}_C2.json | grep "tw::" || true
for c in C1 C2 C3 C5; do
  timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"attn_kernel|quest_select|topp_unit|topp_head|estimate_kernel|quest_filter|append_kernel|merge_kernel|unit_step" -c 8 \
    -o gpurun_out/full_${TAG}_$c python tools/prof_step.py --config $c --reps 1 > /dev/null 2>&1
  python tools/ncu_hot.py gpurun_out/full_${TAG}_$c.ncu-rep . --lines 6 > gpurun_out/ncu_full_${TAG}_$c.txt 2>&1
  python tools/traffic_json.py gpurun_out/full_${TAG}_$c.ncu-rep $c > gpurun_out/traffic_${TAG}_$c.json 2>&1 || true
done
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
