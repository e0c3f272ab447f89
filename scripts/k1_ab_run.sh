#!/bin/bash
# GPU box: K1 / K4 rates (bench.hbm_kernels) of the in-tree library and of abl/*.so variants, interleaved.
# Usage: k1_ab_run.sh OUT name1 name2 ...   ("main" = paper_2501_10709_b200/libfinenv.so)
cd "$(dirname "$0")/.."
out=gpurun_out/$1; shift
for i in 1 2 3; do
  for n in "$@"; do
    if [ "$n" = main ]; then L=$PWD/paper_2501_10709_b200/libfinenv.so; else L=$PWD/abl/$n.so; fi
    echo "$n $(FIN_LIB_PATH=$L timeout 300 python scripts/k1_ab.py 2>&1 | tail -1)" >> $out
  done
done
