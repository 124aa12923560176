#!/bin/bash
# build experiment variants of libspk (timing only) into exp/
mkdir -p exp
for e in "$@"; do
  objs=""
  for f in paper_2301_13659_b200/csrc/*.cu; do
    b=$(basename $f .cu)
    if [ $b = conv_tc ]; then
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSPK_EXP=$e -Xcompiler -fPIC,-fvisibility=hidden -Iinclude -Ipaper_2301_13659_b200/csrc -c $f -o exp/conv_tc_$e.o 2>/dev/null
      objs="$objs exp/conv_tc_$e.o"
    else
      objs="$objs paper_2301_13659_b200/build/$b.o"
    fi
  done
  nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs -o exp/libspk_exp$e.so -cudart static
done
