#!/bin/bash
# Build A/B variants of the library (extra nvcc defines) into
# paper_2011_00162_b200/variants/<name>.so for kernel experiments:
#   scripts/build_variants.sh name1:"-DFOO" name2:"-DBAR" ...
# Select one at run time with PDD_LIB=paper_2011_00162_b200/variants/<name>.so.
set -e
cd "$(dirname "$0")/.."
PKG=paper_2011_00162_b200
mkdir -p $PKG/variants build/variants
for spec in "$@"; do
  name="${spec%%:*}"; defs="${spec#*:}"
  objs=()
  for src in $PKG/csrc/*.cu $PKG/csrc/*.cpp; do
    o=build/variants/$name.$(basename $src).o
    lang=""; [[ $src == *.cpp ]] && lang="-x cu"
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 --expt-relaxed-constexpr \
      -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include -I $PKG/csrc $defs $lang -c $src -o $o &
    objs+=($o)
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $PKG/variants/$name.so "${objs[@]}" -ldl -lpthread
  echo "built $PKG/variants/$name.so"
done
