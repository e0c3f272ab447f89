#!/bin/bash
# One profiling call: full ncu captures (source-mapped) of K3 (fused rollout), K1 and K6.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2501_10709_b200.build > gpurun_out/build.log 2>&1
python scripts/prof_rollout.py 65536 32 2 > gpurun_out/rollout_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:k_tc_rollout" -s 2 -c 1 \
      -o gpurun_out/prof_k3 -f python scripts/prof_rollout.py 65536 32 2 > gpurun_out/ncu_k3.log 2>&1
python scripts/prof_hbm.py k6 > gpurun_out/k6_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:k_pass" -s 3 -c 1 \
      -o gpurun_out/prof_k6 -f python scripts/prof_hbm.py k6 3 > gpurun_out/ncu_k6.log 2>&1
FIN_TIMING=b2b python scripts/prof_hbm.py k1 > gpurun_out/k1_plain.log 2>&1 && \
  FIN_TIMING=b2b ncu --set full --clock-control none --import-source on -k "regex:k_stock_step" -s 10 -c 1 \
      -o gpurun_out/prof_k1 -f python scripts/prof_hbm.py k1 > gpurun_out/ncu_k1.log 2>&1
echo "profile done" >> gpurun_out/summary.txt
