#!/bin/bash
# K4 occupancy experiment: rebuild with FIN_K4_MINB = 2, 3, 4 and time K4 (N = 2^20, T = 32)
cd "$(dirname "$0")/.."
for m in "$@"; do
  FIN_NVCC_FLAGS="-DFIN_K4_MINB=$m" python -m paper_2501_10709_b200.build --force > gpurun_out/build_$m.log 2>&1
  echo "minb=$m $(python scripts/prof_hbm.py k4)" >> gpurun_out/k4_sweep.txt
done
python -m paper_2501_10709_b200.build --force > gpurun_out/build.log 2>&1
