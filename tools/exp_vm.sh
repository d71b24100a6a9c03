timeout 300 ncu --set full --clock-control none --import-source on -k regex:linalg_kernel -c 1 -o gpurun_out/vm1 python tools/prof_sweep.py --kind 2 --reps 2 > gpurun_out/ncu_vm1.log 2>&1
