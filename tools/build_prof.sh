#!/bin/bash
# Builds ab/liblabuf_prof.so: the library with the mode-ii phase timestamps
# (-DLABUF_UT_PROF, read by tools/ut_prof.py).  Run after a normal build.
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
    --expt-relaxed-constexpr -DLABUF_UT_PROF -c -o /tmp/fold_ut_prof.o paper_2605_19049_b200/csrc/fold_ut.cu
mkdir -p ab
cd paper_2605_19049_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../ab/liblabuf_prof.so $(ls *.o | grep -v fold_ut) \
    /tmp/fold_ut_prof.o -ldl -lpthread
