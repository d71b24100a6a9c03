# ncu --set full captures of the non-headline kernels (one launch each), for profiles/
set -x
NCU="timeout 600 ncu --set full --clock-control none --import-source on"
$NCU -k regex:encode_kernel -c 1 -o gpurun_out/p_encode python tools/prof_sweep.py --reps 1 --kind 1 --trees 0 > gpurun_out/p_encode.log 2>&1
$NCU -k regex:index_blocks -c 1 -o gpurun_out/p_index python tools/prof_sweep.py --reps 1 --kind 1 --trees 0 > gpurun_out/p_index.log 2>&1
$NCU -k regex:epoch_cluster -c 1 -o gpurun_out/p_mgd3 python tools/mgd_bench.py --config 3 --rows 200000 --epochs 1 > gpurun_out/p_mgd3.log 2>&1
$NCU -k regex:epoch_large -c 1 -o gpurun_out/p_mgd4 python tools/mgd_bench.py --config 4 --rows 100000 --epochs 1 > gpurun_out/p_mgd4.log 2>&1
$NCU -k regex:mlp_ -c 4 -o gpurun_out/p_mlp python tools/mlp_bench.py --rows 20000 --epochs 1 > gpurun_out/p_mlp.log 2>&1
