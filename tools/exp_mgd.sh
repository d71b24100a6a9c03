timeout 600 python -m pytest tests/test_gpu_training.py -x -q > gpurun_out/t_tr.log 2>&1; echo rc=$? >> gpurun_out/t_tr.log
timeout 600 python tools/mgd_bench.py --config 3 --rows 400000 --epochs 2 > gpurun_out/mgd3_trace.log 2>&1
