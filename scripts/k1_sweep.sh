#!/bin/bash
# K1 occupancy experiment: rebuild with FIN_K1_MINB = 2, 3, 4 and time K1 at N = 2^22
cd "$(dirname "$0")/.."
for m in "$@"; do
  FIN_NVCC_FLAGS="-DFIN_K1_MINB=$m" python -m paper_2501_10709_b200.build --force > gpurun_out/build_$m.log 2>&1
  echo "minb=$m $(python scripts/prof_hbm.py k1)" >> gpurun_out/k1_sweep.txt
done
python -m paper_2501_10709_b200.build --force > gpurun_out/build.log 2>&1
