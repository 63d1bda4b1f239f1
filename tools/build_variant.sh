#!/bin/bash
# Build a variant of the library for A/B timing: tools/build_variant.sh NAME "FILE.cu ..." "-DFLAGS"
# Reuses the regular objects (make first) and recompiles only the listed TUs with the flags.
set -e
cd "$(dirname "$0")/../paper_1707_05141_b200/csrc"
make -s -j8
mkdir -p ../../var_libs build_var_$1
objs=""
for o in build/*.o; do
  src=$(basename ${o%.o}).cu
  if [[ " $2 " == *" $src "* ]]; then
    nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $3 -c $src -o build_var_$1/${src%.cu}.o
    objs="$objs build_var_$1/${src%.cu}.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../var_libs/lib_$1.so $objs -Xcompiler -fvisibility=hidden
rm -rf build_var_$1
echo "built var_libs/lib_$1.so"
