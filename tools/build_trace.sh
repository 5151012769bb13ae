#!/bin/bash
# Trace build of libneo (prefill clock64 stamps) for tools/prefill_trace.py.
cd "$(dirname "$0")/.." && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
  --shared -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr -DNEO_PREFILL_TRACE -I include \
  -o tools/libneo_trace.so paper_2411_01142_b200/csrc/*.cu paper_2411_01142_b200/csrc/*.cpp
