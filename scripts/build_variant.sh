#!/bin/bash
# usage: build_variant.sh NAME "EXTRA_FLAGS"
set -e
name=$1; flags=$2
d=/tmp/var_$name; mkdir -p $d
cd /root/repo/paper_1004_3114_b200/csrc
for f in smem_engine group_engine smem_f32_n2 smem_f32_n4 smem_f64_n2 smem_f64_n4 smem_r64 hbm_engine cluster_engine misc stats_ad baselines reference_api capi; do
  nice nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -fmad=false --extended-lambda -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v -I../../include -I. $flags -c $f.cu -o $d/$f.o 2> $d/$f.log &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../libwrng_gpu_$name.so $d/*.o
grep -A2 "k_smemIfLi4ELi10ELi0ELb1E" $d/smem_f32_n4.log | grep -E "spill|registers"
