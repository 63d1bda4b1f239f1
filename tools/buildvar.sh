#!/bin/bash
# buildvar.sh NAME "DEFINES"
set -e
cd /root/repo/paper_1707_05141_b200/csrc
B=/root/repo/build_var/$1; mkdir -p $B
FL="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $2"
for f in api svd_kernels svd_reg svd_rr qr_kernels qr_reg block_kernels util_kernels; do
  nvcc $FL -fmad=${FMAD:-true} -c $f.cu -o $B/$f.o 2>/dev/null &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/build_var/lib_$1.so $B/*.o -Xcompiler -fvisibility=hidden
echo built $1
