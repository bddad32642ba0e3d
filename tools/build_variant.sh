#!/bin/bash
# Build a variant of libhelr_ckks.so for A/B timing: recompile only the listed
# .cu files with extra -D flags and link them with the default build's objects.
#   tools/build_variant.sh TAG "-DHELR_NTT_EXP=1" ops.cu [ks.cu ...]
# -> paper_2406_13221_b200/libhelr_TAG.so   (select with HELR_LIB=<path>)
set -e
TAG=$1; DEFS=$2; shift 2
PKG=$(dirname "$0")/../paper_2406_13221_b200
mkdir -p $PKG/_obj/var_$TAG
objs=""
for f in $PKG/_obj/*.o; do
  b=$(basename $f .o); use=$f
  for s in "$@"; do [ "$s" = "$b.cu" ] && use=$PKG/_obj/var_$TAG/$b.o; done
  objs="$objs $use"
done
pids=""
for s in "$@"; do
  b=$(basename $s .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 $DEFS \
       -c $PKG/csrc/$s -o $PKG/_obj/var_$TAG/$b.o &
  pids="$pids $!"
done
for p in $pids; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $PKG/libhelr_$TAG.so $objs
echo built $PKG/libhelr_$TAG.so
