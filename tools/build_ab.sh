#!/bin/bash
# Build libsirius.so from git revision $1 into build/ab/libsirius_$2.so (A/B timing via SIRIUS_LIB).
set -e
REV=$1; NAME=$2
D=$(mktemp -d)
git archive "$REV" paper_2409_03856_b200/csrc include | tar -x -C "$D"
mkdir -p build/ab
objs=""
for s in "$D"/paper_2409_03856_b200/csrc/*.cu; do
  o="$D/$(basename "$s").o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -c "$s" -o "$o" &
  objs="$objs $o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/libsirius_$NAME.so $objs -ldl
rm -rf "$D"
echo build/ab/libsirius_$NAME.so
