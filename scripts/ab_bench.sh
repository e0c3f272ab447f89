#!/bin/bash
# A/B the headline bench line over several builds of libfinenv.so (FIN_LIB_PATH), interleaved.
# Usage: ab_bench.sh OUT lib1.so lib2.so ...   (paths relative to the repo root)
cd "$(dirname "$0")/.."
out=gpurun_out/$1; shift
for i in 1 2 3; do
  for L in "$@"; do
    r=$(FIN_LIB_PATH=$PWD/$L python bench.py --no-extras --steps 10 --warmup 3 2>&1 | \
        python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['value'], d['ms_per_step'])")
    echo "$L $r" >> $out
  done
done
