timeout 300 ncu --set full --clock-control none --import-source on -k regex:linalg_kernel -c 1 -o gpurun_out/mv1 python tools/prof_sweep.py --kind 1 --reps 2 > gpurun_out/ncu_mv1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:linalg_kernel -c 1 -o gpurun_out/fused1 python tools/prof_sweep.py --kind 3 --reps 2 > gpurun_out/ncu_fused1.log 2>&1
