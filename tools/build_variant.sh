#!/usr/bin/env bash
# Build an experiment variant of libtadakv_b200.so with extra nvcc defines for ONE source file (others reused
# from build/): tools/build_variant.sh NAME SRC "DEFINES"  ->  variants/NAME/libtadakv_b200.so
# Load it with TADA_LIB_PATH=variants/NAME/libtadakv_b200.so (tools and A/B timing only).
set -eu
name=$1; src=$2; defs=${3:-}
make -s -j8 >/dev/null
mkdir -p variants/$name
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
$NV $defs -c paper_2506_04642_b200/csrc/$src.cu -o variants/$name/$src.o
objs=$(ls build/*.o | grep -v "/$src.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o variants/$name/libtadakv_b200.so \
  $objs variants/$name/$src.o -Xlinker --version-script=paper_2506_04642_b200/csrc/exports.map
echo variants/$name/libtadakv_b200.so
