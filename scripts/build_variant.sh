#!/bin/bash
# Build a variant of libfinenv.so with extra nvcc flags into abl/NAME.so (A/B runs on the GPU box
# with FIN_LIB_PATH=abl/NAME.so).  Usage: build_variant.sh NAME "-DFLAG=1 ..."
cd "$(dirname "$0")/.."
mkdir -p abl
FIN_BUILD_DIR=build/var_$1 FIN_LIB_OUT=abl/$1.so FIN_NVCC_FLAGS="$2" python -m paper_2501_10709_b200.build && rm -rf build/var_$1
