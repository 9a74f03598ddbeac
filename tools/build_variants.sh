#!/bin/bash
# Build engine variants with extra nvcc defines into tools/variants/<name>.so
# usage: tools/build_variants.sh name1 "-DFLAG=1 ..." name2 "..." ...
set -e
ROOT=$(cd $(dirname $0)/.. && pwd)
mkdir -p $ROOT/tools/variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=/tmp/skg_var_$name
  rm -rf $d; mkdir -p $d
  cp -r $ROOT/paper_2502_16949_b200 $d/; cp -r $ROOT/include $d/
  rm -rf $d/paper_2502_16949_b200/build $d/paper_2502_16949_b200/libskge_b200.so
  make -s -j8 -C $d/paper_2502_16949_b200 NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $flags" > /dev/null 2>&1
  cp $d/paper_2502_16949_b200/libskge_b200.so $ROOT/tools/variants/$name.so
  echo built $name
done
