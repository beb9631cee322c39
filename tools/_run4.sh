timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"topp" --csv --log-file gpurun_out/topp_launch.csv python tools/prof_step.py --config C2 --reps 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/topp_launch.csv | head -20
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"topp" -c 2 -o gpurun_out/topp_full python tools/prof_step.py --config C2 --reps 1 > /dev/null 2>&1
python tools/ncu_hot.py gpurun_out/topp_full.ncu-rep . --lines 12 2>&1 | head -60
