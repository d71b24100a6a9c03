timeout 400 python -m pytest tests/test_gpu_linalg.py -x -q > gpurun_out/t_linalg.log 2>&1; echo rc=$? >> gpurun_out/t_linalg.log
for sp in 0 1; do for k in 1 2 3; do
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:linalg_kernel -c 1 python tools/prof_sweep.py --kind $k --reps 2 --splits $sp > gpurun_out/exp_sp${sp}_k$k.log 2>&1
done; done
