#!/bin/bash
# Experiment builds of the bf16 flat kernels with one prologue/epilogue piece
# compiled out (NVRAR_ABL_* in csrc/nvrar_kernels.cuh), linked with the other
# objects of the product build; load one with NVRAR_LIB=build_exp/<name>/libnvrar_b200.so.
# Measurement only: the ablations break the call sequence for P > 1.
set -e
cd "$(dirname "$0")/.."
LIB=paper_2511_09557_b200/lib
for v in NO_SEQ NO_END NO_SYNC2; do
  d=build_exp/$v; mkdir -p $d
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --fmad=false -cudart static -Iinclude -DNVRAR_ABL_$v -c paper_2511_09557_b200/csrc/nvrar_flat_bf16.cu -o $d/nvrar_flat_bf16.o &
done
wait
for v in NO_SEQ NO_END NO_SYNC2; do
  d=build_exp/$v
  objs=$(ls $LIB/*.o | grep -v nvrar_flat_bf16.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/libnvrar_b200.so $objs $d/nvrar_flat_bf16.o
done
ls -la build_exp/*/libnvrar_b200.so
