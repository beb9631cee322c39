ncu --set full --import-source on --clock-control none -k regex:'append_kernel|quest_filter|quest_select|estimate_kernel|topp_head|attn_kernel|merge_kernel' -c 8 -o gpurun_out/step_c2 -f python tools/prof_step.py --config C2 --reps 1 > gpurun_out/ncu_step.log 2>&1
ls -la gpurun_out/step_c2.ncu-rep
