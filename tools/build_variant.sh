#!/bin/bash
# Build an A/B variant of libmpm.so for tools/time_step.py:
#   tools/build_variant.sh <name> [git-rev|-] [-DMACRO=V ...]
# "-" (default) builds the working tree; a git revision builds that commit's sources.
# Output: paper_1810_01054_b200/libmpm_<name>.so (git-ignored; travels with gpurun).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
rev=${1:--}; [ $# -gt 0 ] && shift
src=$ROOT
if [ "$rev" != "-" ]; then
  src=$(mktemp -d)
  mkdir -p "$src/include" "$src/paper_1810_01054_b200/csrc"
  for f in include/mpm.h paper_1810_01054_b200/csrc/mpm_api.cu paper_1810_01054_b200/csrc/mpm_kernels.cuh; do
    git -C "$ROOT" show "$rev:$f" > "$src/$f"
  done
fi
cd "$src/paper_1810_01054_b200/csrc"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared "$@" -o "$ROOT/paper_1810_01054_b200/libmpm_$name.so" mpm_api.cu -ldl
