#!/bin/bash
# Build an experimental variant of the library: tools/abl_build.sh NAME [-DFOO=1 ...]
# Output tools/abl/NAME.so (git-ignored; travels to the GPU box); select it with AMS_LIB.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p tools/abl
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo \
  -Xcompiler -fPIC,-O3 -shared --expt-relaxed-constexpr -I include "$@" \
  paper_1410_6754_b200/csrc/*.cu paper_1410_6754_b200/csrc/host/*.cpp -o tools/abl/$name.so
echo tools/abl/$name.so
