#!/bin/bash
# Build A/B variants of the library with extra nvcc flags into _lib_ab/<tag>/ (local, no GPU):
#   bash tools/ab_variants.sh tag1 "-DX=1" tag2 "-DY=2" ...
set -e
while [ $# -ge 2 ]; do
  tag=$1; flags=$2; shift 2
  mkdir -p _lib_ab/$tag
  TH_EXTRA_NVCC_FLAGS="$flags" python -m paper_2504_15814_b200.build --force --out $PWD/_lib_ab/$tag/libtrihalo_b200.so > /dev/null 2>&1 &
done
wait
ls -la _lib_ab/*/libtrihalo_b200.so
