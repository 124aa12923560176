# conv1 bottleneck localisation: timing-experiment variants + role clocks (C2)
mkdir -p gpurun_out; rm -f gpurun_out/ab_conv1.txt
SPK_PREC=auto timeout 120 python scripts/time_conv.py c2 base >> gpurun_out/ab_conv1.txt 2>&1
for v in e32 e128 e4096 e160 e6 e4256; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 60 python scripts/time_conv.py c2 $v >> gpurun_out/ab_conv1.txt 2>&1 || echo "$v fail" >> gpurun_out/ab_conv1.txt; done
SPK_LIB_OVERRIDE=exp/libspk_prof.so timeout 120 python scripts/prof_conv.py c2 >> gpurun_out/ab_conv1.txt 2>&1
