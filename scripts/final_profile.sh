#!/bin/bash
# Round-end evidence: launch list of the bench command, ncu --set full of the bench's own
# rollout launch (traffic for bench.py's roofline), of K3 at T = 32, K1, K6 and the GAE pass.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2501_10709_b200.build > gpurun_out/build.log 2>&1
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_tc_rollout" -s 3 -c 1 \
    -o gpurun_out/prof_bench -f python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_tc_rollout" -s 2 -c 1 \
    -o gpurun_out/prof_k3 -f python scripts/prof_rollout.py 65536 32 2 > gpurun_out/ncu_k3.log 2>&1
FIN_TIMING=b2b ncu --set full --clock-control none --import-source on -k "regex:k_stock_step" -s 10 -c 1 \
    -o gpurun_out/prof_k1 -f python scripts/prof_hbm.py k1 > gpurun_out/ncu_k1.log 2>&1
FIN_TIMING=b2b ncu --set full --clock-control none --import-source on -k "regex:k_stock_replay" -s 10 -c 1 \
    -o gpurun_out/prof_k4 -f python scripts/prof_hbm.py k4 > gpurun_out/ncu_k4.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_metrics" -s 3 -c 1 \
    -o gpurun_out/prof_k6 -f python scripts/prof_hbm.py k6 3 > gpurun_out/ncu_k6.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_gae_tma" -s 2 -c 1 \
    -o gpurun_out/prof_gae -f python scripts/gae_prof.py > gpurun_out/ncu_gae.log 2>&1
echo "final profile done" >> gpurun_out/summary.txt
