#!/bin/bash
# tools/build_variant.sh NAME [OBG_CU]: compile a variant of obg.cu into _ab/NAME/libobg.so
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
SRC=${2:-$REPO/paper_1412_1945_b200/csrc/obg.cu}
mkdir -p "$REPO/_ab/$1"
cp "$SRC" "$REPO/_ab/$1/obg.cu"
cp "$REPO/paper_1412_1945_b200/csrc/obg_io.cpp" "$REPO/_ab/$1/"
cd "$REPO/_ab/$1"
nvcc $NVEXTRA -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --shared \
  -I"$REPO/paper_1412_1945_b200/csrc" -o libobg.so obg.cu obg_io.cpp 2> ptxas.log || (cat ptxas.log; false)
