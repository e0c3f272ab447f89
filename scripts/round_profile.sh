#!/bin/bash
# One GPU call: gpu tests, smoke, bench, then ncu (launch list of the bench command +
# full captures of the fused rollout K3, the step kernel K1 and the metrics pass K6).
# Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/gpu_tests.sh tests/test_gpu_env.py tests/test_gpu_policy.py tests/test_gpu_metrics.py \
  tests/test_gpu_ensemble.py tests/test_gpu_market.py
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?" >> gpurun_out/summary.txt
python bench.py > gpurun_out/bench.log 2>&1; echo "bench $?" >> gpurun_out/summary.txt
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_launch.log 2>&1
python scripts/prof_rollout.py 65536 32 2 > gpurun_out/rollout_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:k_tc_rollout" -s 2 -c 1 \
      -o gpurun_out/prof_k3 -f python scripts/prof_rollout.py 65536 32 2 > gpurun_out/ncu_k3.log 2>&1
FIN_TIMING=b2b python scripts/prof_hbm.py k1 > gpurun_out/k1_plain.log 2>&1 && \
  FIN_TIMING=b2b ncu --set full --clock-control none --import-source on -k "regex:k_stock_step" -s 10 -c 1 \
      -o gpurun_out/prof_k1 -f python scripts/prof_hbm.py k1 > gpurun_out/ncu_k1.log 2>&1
python scripts/prof_hbm.py k6 > gpurun_out/k6_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:k_metrics" -s 3 -c 1 \
      -o gpurun_out/prof_k6 -f python scripts/prof_hbm.py k6 3 > gpurun_out/ncu_k6.log 2>&1
echo "profile done" >> gpurun_out/summary.txt
