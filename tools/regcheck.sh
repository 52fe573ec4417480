#!/bin/bash
# Compile-only register check of one solve-kernel instantiation (~12 s):
#   tools/regcheck.sh [float|double] [kernels.cuh]
# prints ptxas' spill line for solve_kernel<W,1,false> and the number of
# local-memory instructions (LDL/STL) in its SASS.
W=${1:-float}
SRC=${2:-$(dirname "$0")/../paper_2011_01850_b200/csrc/gmres_kernels.cuh}
D=$(mktemp -d)
cp "$SRC" "$D/gmres_kernels.cuh"
printf '#include "gmres_kernels.cuh"\nvoid* p[] = {(void*)&g200::solve_kernel<%s, %s, false>};\n' "$W" "${L:-1}" > "$D/one.cu"
/usr/local/cuda/bin/nvcc -Xptxas=-v -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -c -o "$D/one.o" "$D/one.cu" 2>&1 \
  | grep -A1 "Function properties for _ZN4g20012solve_kernel" | grep spill
echo "LDL/STL: $(cuobjdump -sass "$D/one.o" | grep -c 'LDL\|STL')"
rm -rf "$D"
