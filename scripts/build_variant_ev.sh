#!/bin/bash
# build libspk with an alternative conv_event.cu (A/B timing on one box): build_variant_ev.sh NAME SRC.cu ["-DFLAGS"]
set -e
mkdir -p exp
objs=""
for f in paper_2301_13659_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  if [ $b = conv_event ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 $3 -Xcompiler -fPIC,-fvisibility=hidden -Iinclude -Ipaper_2301_13659_b200/csrc -c $2 -o exp/conv_event_$1.o
    objs="$objs exp/conv_event_$1.o"
  else
    objs="$objs paper_2301_13659_b200/build/$b.o"
  fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs -o exp/libspk_$1.so -cudart static
