timeout 600 python -m pytest tests/test_gpu_topp.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in C2 C5 C3; do timeout 300 python tools/stage_time.py --config $c --layers 1 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"topp" --csv --log-file gpurun_out/topp_launch.csv python tools/prof_step.py --config C2 --reps 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/topp_launch.csv | head -20
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"topp" -c 3 -o gpurun_out/topp_full python tools/prof_step.py --config C2 --reps 1 > /dev/null 2>&1
python tools/ncu_hot.py gpurun_out/topp_full.ncu-rep . --lines 14 2>&1 | head -80
