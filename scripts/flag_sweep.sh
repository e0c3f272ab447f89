#!/bin/bash
# Rebuild with each set of nvcc -D flags and run a command, appending its output.
# Usage: flag_sweep.sh OUT "command" "-DFLAGS1" "-DFLAGS2" ...   (OUT under gpurun_out/)
cd "$(dirname "$0")/.."
out=gpurun_out/$1; cmd=$2; shift 2
for f in "$@"; do
  FIN_NVCC_FLAGS="$f" python -m paper_2501_10709_b200.build --force > gpurun_out/build_sweep.log 2>&1
  echo "== $f" >> $out
  bash -c "$cmd" >> $out 2>&1
done
python -m paper_2501_10709_b200.build --force > gpurun_out/build.log 2>&1
