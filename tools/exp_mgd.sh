timeout 600 python -m pytest tests/test_gpu_training.py -x -q > gpurun_out/t_tr.log 2>&1; echo rc=$? >> gpurun_out/t_tr.log
for i in 1 2; do timeout 600 python tools/mgd_bench.py --config 3 --epochs 3 > gpurun_out/mgd3_full_$i.log 2>&1; done
