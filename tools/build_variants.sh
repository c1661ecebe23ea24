#!/bin/bash
# Build experiment variants of the engine library into variants/ (git-ignored,
# travels to the GPU box).  Usage: tools/build_variants.sh NAME "-DFLAG=1 ..." ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/variants"
C="$ROOT/paper_2112_02958_b200/csrc"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC --expt-relaxed-constexpr $flags -shared -I "$ROOT/include" -I "$C" \
    "$C/pe_engine.cu" "$C/pe_graph.cc" "$C/pe_pir.cc" "$C/pe_search.cc" "$C/pe_nccl.cc" -ldl -o "$ROOT/variants/$name.so" &
done
wait
