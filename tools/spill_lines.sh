#!/bin/bash
# Source lines of the local-memory (spill) instructions of one solve-kernel instantiation:
#   tools/spill_lines.sh [float|double] [L] [extra template args, e.g. ", false, true" for the chunk-ring kernel]
W=${1:-float}
L=${2:-1}
EXTRA=${3:-}
SRC=$(dirname "$0")/../paper_2011_01850_b200/csrc/gmres_kernels.cuh
D=$(mktemp -d)
cp "$SRC" "$D/gmres_kernels.cuh"
printf '#include "gmres_kernels.cuh"\nvoid* p[] = {(void*)&g200::solve_kernel<%s, %s, false%s>};\n' "$W" "$L" "$EXTRA" > "$D/one.cu"
/usr/local/cuda/bin/nvcc -lineinfo -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -cubin -o "$D/one.cubin" "$D/one.cu"
/usr/local/cuda/bin/nvdisasm -g -c "$D/one.cubin" | awk '/\/\/## File/ {loc=$0} /LDL|STL/ {print loc}' \
  | sed -E 's/.*line ([0-9]+).*/\1/' | sort -n | uniq -c
rm -rf "$D"
