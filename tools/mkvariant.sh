#!/bin/bash
# usage: mkvar.sh name "extra flags"
set -e
name=$1; shift
out=/root/repo/build_variants/$name; mkdir -p $out
cd /root/repo/paper_2008_11480_b200/csrc
objs=""
for f in gemm_tma kernels engine steps batched peer setup shard capi; do
  if [ "$f" = batched ] || [ ! -f build/$f.o ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden $@ -c $f.cu -o $out/$f.o &
    objs="$objs $out/$f.o"
  else objs="$objs build/$f.o"; fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libseriesinv_b200.so $objs -lcudart -ldl
echo built $out
