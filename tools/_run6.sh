timeout 600 ncu --set full --import-source on --clock-control none -k regex:"topp_hist|topp_resolve" -c 2 -o gpurun_out/topp_full3 python tools/prof_step.py --config C2 --reps 1 > /dev/null 2>&1
