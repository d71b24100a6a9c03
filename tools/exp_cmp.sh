for i in 1 2; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:levels_kernel -c 1 python tools/prof_sweep.py --levels 1 --reps 2 --kind 3 > gpurun_out/cmp_lv$i.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:linalg_kernel -c 1 python tools/prof_sweep.py --reps 2 --kind 3 > gpurun_out/cmp_tc$i.log 2>&1
done
python tools/prof_sweep.py --levels 1 --reps 1 --kind 3 > gpurun_out/cmp_size.log 2>&1
