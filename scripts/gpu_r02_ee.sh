# C5 conv1/conv2 share of the fire epilogue (x128: no epilogue work) and of the MMAs (x32)
mkdir -p gpurun_out/ee
for v in base x128 x32; do
  if [ $v = base ]; then SPK_PREC=auto timeout 300 python scripts/time_conv.py c5 base >> gpurun_out/ee/conv.txt 2>&1
  else SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py c5 $v >> gpurun_out/ee/conv.txt 2>&1; fi
done
