#!/bin/bash
# Builds ab/liblabuf_ckprof.so: the library with the per-CTA timeline of the
# bf16 state-kind chunk kernel (-DLABUF_CK_PROF, read by tools/ck_prof.py).
set -e
for f in chunk_bf16_state chunk_bf16h_direct; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
    --expt-relaxed-constexpr -DLABUF_CK_PROF -c -o /tmp/${f}_prof.o paper_2605_19049_b200/csrc/$f.cu &
done
wait
mkdir -p ab
cd paper_2605_19049_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../ab/liblabuf_ckprof.so $(ls *.o | grep -v "chunk_bf16_state\|chunk_bf16h_direct") \
    /tmp/chunk_bf16_state_prof.o /tmp/chunk_bf16h_direct_prof.o -ldl -lpthread
