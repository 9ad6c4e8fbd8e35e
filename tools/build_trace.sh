#!/bin/bash
# Debug build of the CUDA library with clock64 pipeline stamps (-DPA_TRACE) -> tools/libpa_trace.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build_trace
for f in paper_2507_04239_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DPA_TRACE $EXTRA \
    -c "$f" -o build_trace/$(basename "$f").o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libpa_trace.so build_trace/*.o
