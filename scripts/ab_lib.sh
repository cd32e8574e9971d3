#!/bin/bash
# Build build/ab/libdicm_b200_<rev>.so: the current objects with ONE source
# file taken from git revision <rev> (default HEAD), for same-box A/B runs via
# DICM_LIB_PATH.  Usage: bash scripts/ab_lib.sh paper_1711_06505_b200/csrc/sample.cu [rev]
set -e
src=$1; rev=${2:-HEAD}
cd "$(dirname "$0")/.."
make -s -j 16
mkdir -p build/ab
base=$(basename "$src" .cu)
git show "$rev:$src" > build/ab/${base}_${rev}.cu
cp paper_1711_06505_b200/csrc/*.cuh build/ab/
/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I include -I paper_1711_06505_b200/csrc -c build/ab/${base}_${rev}.cu -o build/ab/${base}_${rev}.o
objs=$(ls build/obj/*.o | grep -v "/${base}.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -pthread \
  -o build/ab/libdicm_b200_${rev}.so $objs build/ab/${base}_${rev}.o
echo build/ab/libdicm_b200_${rev}.so
