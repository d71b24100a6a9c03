timeout 900 python -m pytest tests/test_gpu_training.py -x -q > gpurun_out/t_c16.log 2>&1; echo rc=$? >> gpurun_out/t_c16.log
timeout 600 python tools/mgd_bench.py --config 4 --epochs 3 > gpurun_out/mgd4_full.log 2>&1
timeout 600 python tools/mgd_bench.py --config 4 --epochs 3 --dsmem > gpurun_out/mgd4_full_dsmem.log 2>&1
