#!/bin/bash
# Build libmbe.so with extra -D defines into variants/<name>.so (A/B timing via MBE_LIB_PATH).
#   scripts/build_variant.sh <name> [DEFINE=VALUE ...] [-Xptxas=-O2 ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants
defs=""; for d in "$@"; do case "$d" in -*) defs="$defs ${d/=/ }";; *) defs="$defs -D$d";; esac; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC,-O2 \
  $defs -I include -o variants/$name.so paper_2401_05039_b200/csrc/*.cu
echo variants/$name.so
