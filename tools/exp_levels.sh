# level-kernel iteration: GPU parity, a short bench, one ncu capture
timeout 400 python -m pytest tests/test_gpu_linalg.py -x -q > gpurun_out/t_linalg.log 2>&1; echo rc=$? >> gpurun_out/t_linalg.log
timeout 300 python bench.py --no-mgd --no-cpu-baseline --steps 50 > gpurun_out/bench_lv.json 2> gpurun_out/bench_lv.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:levels_kernel -c 1 -o gpurun_out/lv${1:-x} python tools/prof_sweep.py --levels 1 --reps 2 > gpurun_out/ncu_lv.log 2>&1
