for m in 0 3 1; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:levels_kernel -c 1 python tools/prof_sweep.py --levels 1 --reps 2 --prefetch $m > gpurun_out/exp_pf$m.log 2>&1
done
