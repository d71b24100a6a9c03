# headline evidence at the current build: ncu launch list of the bench command, one full capture of the
# slot-cache kernel (fused), the per-batch phase trace
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:levels_kernel -c 1 -o gpurun_out/p_slots_k3 python tools/prof_sweep.py --kind 3 --reps 2 --levels 1 > gpurun_out/ncu_headline.log 2>&1
python tools/slots_trace.py > gpurun_out/slots_trace.log 2>&1
