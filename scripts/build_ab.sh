#!/bin/bash
# Build the library of git revision $1 (default HEAD) as paper_1801_09866_b200/librnnlm_a.so
# (the A side of scripts/ab_lib.sh); the working tree's build stays librnnlm.so.
set -eu
rev=${1:-HEAD}
cd "$(dirname "$0")/.."
tmp=$(mktemp -d)
git archive "$rev" paper_1801_09866_b200/csrc include | tar -x -C "$tmp"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared \
  -I"$tmp/include" -o paper_1801_09866_b200/librnnlm_a.so "$tmp"/paper_1801_09866_b200/csrc/*.cu
rm -rf "$tmp"
