#!/bin/bash
# timing variants of the library with RING_SKIP bits (tools/_ringvar, not product code)
cd "$(dirname "$0")/.."
for v in "$@"; do
  /usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
    -Xcompiler -fPIC -cudart static --expt-relaxed-constexpr -DRING_SKIP=$(echo $v | tr -d vp) $( [[ $v == *v ]] && echo -DRING_VSTORE=1 ) $( [[ $v == *p ]] && echo -DRING_PROF=1 ) \
    -o tools/_ringvar/libhygro_skip$v.so paper_1703_10119_b200/csrc/hyg_api.cu paper_1703_10119_b200/csrc/hyg_scaling.cpp &
done
wait
