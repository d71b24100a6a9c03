timeout 900 python -m pytest tests/test_gpu_linalg.py -x -q > gpurun_out/t_terms.log 2>&1; echo rc=$? >> gpurun_out/t_terms.log
for t in 0 1 0 1; do TERMS=$t timeout 300 python tools/sweep_time.py >> gpurun_out/terms_time.log 2>&1; done
