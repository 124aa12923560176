# conv_tc timing switches on the current tree (per-layer ms, C2): which role bounds conv1
mkdir -p gpurun_out/s
for r in 1 2; do
  SPK_PREC=auto timeout 120 python scripts/time_conv.py c2 base >> gpurun_out/s/conv.txt 2>&1
  for v in 32 128 160 4096 2 4 64 512 1024 65536 256; do
    SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_x$v.so timeout 60 python scripts/time_conv.py c2 x$v >> gpurun_out/s/conv.txt 2>&1 || echo "x$v fail" >> gpurun_out/s/conv.txt
  done
done
