#!/bin/bash
# Build an A/B variant of libralpb200.so: recompile one source with extra defines on top of
# the current in-tree objects and link abtest/<name>.so.
# usage: tools/build_variant.sh <name> <source.cu> "<nvcc defines>"
set -e
NAME=$1; SRC=$2; DEFS=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=$ROOT/paper_1901_05803_b200/build
D=$ROOT/abtest/${NAME}_objs
mkdir -p "$D"; cp "$B"/*.o "$D"/
STEM=$(basename "$SRC" .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I "$ROOT/include" $DEFS -c "$ROOT/paper_1901_05803_b200/csrc/$SRC" -o "$D/$STEM.o"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$ROOT/abtest/$NAME.so" "$D"/*.o \
  -lcudart_static -ldl -lrt -lpthread
rm -rf "$D"
echo "$ROOT/abtest/$NAME.so"
