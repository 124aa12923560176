#!/bin/bash
# build libspk with one translation unit replaced (A/B timing): build_variant_any.sh NAME UNIT SRC.cu ["-DFLAGS"]
set -e
mkdir -p exp
objs=""
for f in paper_2301_13659_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  if [ $b = $2 ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 $4 -Xcompiler -fPIC,-fvisibility=hidden -Iinclude -Ipaper_2301_13659_b200/csrc -c $3 -o exp/${2}_$1.o
    objs="$objs exp/${2}_$1.o"
  else
    objs="$objs paper_2301_13659_b200/build/$b.o"
  fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs -o exp/libspk_$1.so -cudart static
