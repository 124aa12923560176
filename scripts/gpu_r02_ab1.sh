# upper bound of offloading one N tile in four of the epilogue work: the epilogue skips its work on nt == 1 tiles (skip1)
mkdir -p gpurun_out/ab1
for r in 1 2 3; do for v in base0 skip1; do
  SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py c2 $v >> gpurun_out/ab1/conv.txt 2>&1 || echo "$v fail" >> gpurun_out/ab1/conv.txt
done; done
