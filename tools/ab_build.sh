#!/bin/bash
# A/B build of libneo with extra defines on neo_prefill.cu only (other objects cached):
#   tools/ab_build.sh <tag> [-DNAME=VAL ...]  ->  tools/libneo_<tag>.so  (NEO_LIB=... selects it)
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr -I include"
mkdir -p /tmp/ab
for f in paper_2411_01142_b200/csrc/*.cu paper_2411_01142_b200/csrc/*.cpp; do
  b=$(basename $f); [ "$b" = neo_prefill.cu ] && continue
  o=/tmp/ab/$b.o
  if [ ! -f $o ] || [ $f -nt $o ] || [ paper_2411_01142_b200/csrc/neo_internal.cuh -nt $o ]; then $NV -c -o $o $f; fi
done
$NV "$@" -c -o /tmp/ab/prefill_$tag.o paper_2411_01142_b200/csrc/neo_prefill.cu
$NV --shared -o tools/libneo_$tag.so /tmp/ab/prefill_$tag.o $(ls /tmp/ab/*.o | grep -v '/prefill_')
echo tools/libneo_$tag.so
