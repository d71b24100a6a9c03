# round-end: full bench line, launch list of the same command, ncu of the headline and the config-4 epoch
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_launch.log 2>&1
NCU="timeout 600 ncu --set full --clock-control none --import-source on"
$NCU -k regex:linalg_kernel -c 1 -o gpurun_out/headline python tools/prof_sweep.py --kind 3 --reps 2 > gpurun_out/ncu_headline.log 2>&1
$NCU -k regex:epoch_large -c 1 -o gpurun_out/p_mgd4 python tools/mgd_bench.py --config 4 --rows 100000 --epochs 1 > gpurun_out/p_mgd4.log 2>&1
