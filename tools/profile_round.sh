#!/bin/bash
# One profiling pass for profiles/: launch list (per-kernel device time + DRAM
# bytes, serialized/cold) and an ncu --set full capture of the hot kernels.
# usage (on the GPU box): tools/profile_round.sh <tag> [config]
set -u
TAG=${1:-r01}
CFG=${2:-C2}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv python tools/prof_step.py --config $CFG --reps 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_${TAG}_${CFG}.csv --json gpurun_out/launches_${TAG}_${CFG}.json | grep "tw::" || true
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"attn_kernel|quest_select|topp_head|estimate_kernel|quest_filter|append_kernel|merge_kernel" -c 8 \
  -o gpurun_out/full_${TAG}_${CFG} python tools/prof_step.py --config $CFG --reps 1 > /dev/null 2>&1
python tools/ncu_hot.py gpurun_out/full_${TAG}_${CFG}.ncu-rep . --lines 6 > gpurun_out/full_${TAG}_${CFG}.txt 2>&1
cat gpurun_out/full_${TAG}_${CFG}.txt | grep -E "^==|time|stalls"
