#!/bin/bash
# Dev A/B: build the library of a git revision: scripts/build_rev.sh NAME REV ["-DFOO"] -> build_variants/NAME/libdfb200.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; REV=$2; shift 2
TMP=$(mktemp -d)
git -C $ROOT archive $REV paper_2601_20499_b200/csrc include | tar -x -C $TMP
OUT=$ROOT/build_variants/$NAME
mkdir -p $OUT
cd $TMP/paper_2601_20499_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I../../include -I. --expt-relaxed-constexpr $*"
for s in df_attn.cu df_kv.cu df_proj.cu; do /usr/local/cuda/bin/nvcc $F -c $s -o $OUT/$s.o & done
/usr/local/cuda/bin/nvcc $F -x cu -c df_host.cpp -o $OUT/df_host.cpp.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC -o $OUT/libdfb200.so $OUT/*.o
rm -rf $TMP
echo built $OUT/libdfb200.so from $REV
