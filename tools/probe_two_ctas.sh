#!/bin/bash
# Probe: would two CTAs per SM hide the slot kernel's phase latencies?  Builds a second library whose
# slot kernels use 512-thread CTAs, two per SM (the cache cut for 512 ranges), and times both
# libraries over config-2 batches cut to their first 392 columns (tables small enough for two CTAs).
# Run from the repo root on the GPU box; the probe library is not part of the product.
set -e
cd paper_1702_06943_b200/csrc
make -s BUILD=build_probe LIB=../libtoc_probe.so EXTRA="-DTOC_LVL_THREADS=512 -DTOC_LVL_CTAS_PER_SM=2" all
cd ../..
python tools/probe_two_ctas.py paper_1702_06943_b200/libtoc_b200.so paper_1702_06943_b200/libtoc_probe.so
