#!/bin/bash
# K1 configuration experiment: rebuild with each set of nvcc -D flags and time K1 at
# N = 2^22 (back-to-back launches).  Usage: k1_sweep.sh "-DFIN_K1_E=1" "-DFIN_K1_E=2" ...
cd "$(dirname "$0")/.."
for f in "$@"; do
  FIN_NVCC_FLAGS="$f" python -m paper_2501_10709_b200.build --force > gpurun_out/build_sweep.log 2>&1
  echo "$f $(FIN_TIMING=b2b python scripts/prof_hbm.py k1)" >> gpurun_out/k1_sweep.txt
done
python -m paper_2501_10709_b200.build --force > gpurun_out/build.log 2>&1
