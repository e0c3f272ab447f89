#!/bin/bash
# K6 configuration experiment: rebuild with each set of nvcc -D flags and time the
# fused metrics pass at T = 2048, N = 2^18.  Usage: k6_sweep.sh "-DFIN_K6_MINB=4" ...
cd "$(dirname "$0")/.."
for f in "$@"; do
  FIN_NVCC_FLAGS="$f" python -m paper_2501_10709_b200.build --force > gpurun_out/build_sweep.log 2>&1
  echo "$f $(python scripts/prof_hbm.py k6)" >> gpurun_out/k6_sweep.txt
done
python -m paper_2501_10709_b200.build --force > gpurun_out/build.log 2>&1
