#!/bin/sh
# developer build: only the bench configuration's instances (f=16, b=16, xor) -> libckf.so
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-O2 -shared -DCKF_DEV_MIN -o paper_2603_15486_b200/libckf.so paper_2603_15486_b200/csrc/ckf_kernels.cu
