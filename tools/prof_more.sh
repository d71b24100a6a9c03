# ncu --set full captures beside the headline: the slot kernel for A.v alone and v^T.A alone, and the fp32 slot kernel (its first launch: A.v alone)
NCU="timeout 600 ncu --set full --clock-control none --import-source on"
$NCU -k regex:levels_kernel -c 1 -o gpurun_out/p_slots_k1 python tools/prof_sweep.py --kind 1 --reps 2 --levels 1 > gpurun_out/ncu_k1.log 2>&1
$NCU -k regex:levels_kernel -c 1 -o gpurun_out/p_slots_k2 python tools/prof_sweep.py --kind 2 --reps 2 --levels 1 > gpurun_out/ncu_k2.log 2>&1
$NCU -k regex:levels32_kernel -c 1 -o gpurun_out/p_slots32_k1 python tools/slots32_time.py > gpurun_out/ncu_s32.log 2>&1
ls -la gpurun_out/*.ncu-rep
