timeout 400 python -m pytest tests/test_gpu_linalg.py -x -q > gpurun_out/t_linalg.log 2>&1; echo rc=$? >> gpurun_out/t_linalg.log
for k in 1 2 3; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:levels_kernel -c 1 python tools/prof_sweep.py --levels 1 --reps 2 --kind $k > gpurun_out/exp_lv_k$k.log 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:linalg_kernel -c 1 python tools/prof_sweep.py --reps 2 --kind 3 > gpurun_out/exp_tc_k3.log 2>&1
python tools/prof_sweep.py --levels 1 --reps 1 --kind 3 > gpurun_out/exp_size.log 2>&1
