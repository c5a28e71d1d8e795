#!/bin/bash
# Build libgim.so from a committed revision into build/libgim_<name>.so (A/B on the GPU box):
#   tools/build_rev.sh HEAD a_head
set -e
REV=${1:-HEAD}; NAME=${2:-rev}
D=build/rev_$NAME
rm -rf $D; mkdir -p $D/csrc $D/../include
for f in $(git ls-tree --name-only $REV paper_2009_07325_b200/csrc/); do git show $REV:$f > $D/csrc/$(basename $f); done
git show $REV:include/gim.h > build/include/gim.h
/usr/local/cuda/bin/nvcc -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -shared -o build/libgim_$NAME.so $D/csrc/*.cu
echo build/libgim_$NAME.so
