# A/B of two builds of the cluster epochs: tools/alt/libtoc_b200.so (ALT) vs the in-tree library (NEW),
# config 3 (step images) and config 4 (part images)
run_alt() { timeout 600 python -c "import sys; sys.argv=['mgd_bench.py','--config','$3','--epochs','3']; sys.path.insert(0,'.'); import paper_1702_06943_b200._native as N; N.LIB_PATH='$1'; exec(open('tools/mgd_bench.py').read(), {'__file__': 'tools/mgd_bench.py', '__name__': '__main__'})" 2>&1 | grep -E "untraced|cluster 8 phase" | sed "s|^|$2 cfg$3 |" >> gpurun_out/ab3.log; }
timeout 600 python -m pytest tests/test_gpu_training.py -x -q > gpurun_out/t_tr.log 2>&1; echo rc=$? >> gpurun_out/t_tr.log
for i in 1 2; do
  for c in 3 4; do
    run_alt tools/alt/libtoc_b200.so ALT $c
    run_alt paper_1702_06943_b200/libtoc_b200.so NEW $c
  done
done
