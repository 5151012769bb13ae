#!/bin/bash
# Host-side sanitizer run (development aid): builds libneo with AddressSanitizer +
# UndefinedBehaviorSanitizer on the host code (pool allocator, swap validation,
# planner, scheduler, CPU attention and its worker pool; nvcc passes the flags to
# g++ for the host side) and runs the CPU test suite against it.
#   bash tools/asan_cpu_suite.sh > profiles/rNN_asan_ubsan.txt 2>&1
set -u
cd "$(dirname "$0")/.."
OUT=tools/libneo_asan.so
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O1 -g -std=c++17 --shared \
  -Xcompiler -fPIC,-fvisibility=hidden,-fsanitize=address,-fsanitize=undefined,-fno-omit-frame-pointer,-fno-sanitize-recover=undefined \
  --expt-relaxed-constexpr -I include -o $OUT paper_2411_01142_b200/csrc/*.cu paper_2411_01142_b200/csrc/*.cpp \
  -Xlinker -lasan -Xlinker -lubsan || exit 1
echo "built $OUT"
PRE="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)"
LD_PRELOAD="$PRE" NEO_LIB=$OUT ASAN_OPTIONS=detect_leaks=0,protect_shadow_gap=0,halt_on_error=1 \
  UBSAN_OPTIONS=print_stacktrace=1,halt_on_error=1 \
  python -m pytest tests -m "not gpu" -q -p no:cacheprovider -x \
  tests/test_abi.py tests/test_cpu_attn.py tests/test_scheduler.py tests/test_bench_harness.py 2>&1 | tail -15
echo "exit=${PIPESTATUS[0]}"
