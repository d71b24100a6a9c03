timeout 900 python -m pytest tests/test_gpu_training.py -x -q > gpurun_out/t_c16.log 2>&1; echo rc=$? >> gpurun_out/t_c16.log
for c in 8 16; do timeout 600 python tools/mgd_bench.py --config 3 --rows 400000 --epochs 2 --cluster $c > gpurun_out/mgd3_c$c.log 2>&1; done
