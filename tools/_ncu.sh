ncu --set full --import-source on --clock-control none -k regex:topp_head -c 1 -o gpurun_out/topp_old -f env TW_LIB_PATH=tools/_variants/minb2/libtwilight.so python tools/prof_step.py --config C2 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:topp_head -c 1 -o gpurun_out/topp_new -f env TW_LIB_PATH=tools/_variants/new_m2/libtwilight.so python tools/prof_step.py --config C2 --reps 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
