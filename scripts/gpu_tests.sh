#!/bin/bash
# Run the -m gpu suites in order of risk; each under its own timeout.
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -m paper_2501_10709_b200.build > gpurun_out/build.log 2>&1
for f in "$@"; do
  n=$(basename "$f" .py)
  timeout 600 python -m pytest "$f" -m gpu -q -x --timeout 180 --timeout-method=thread -p no:cacheprovider \
     > gpurun_out/$n.log 2>&1
  echo "$f exit $?" >> gpurun_out/summary.txt
done
