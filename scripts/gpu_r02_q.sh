# conv1 decomposition on the current tree: timing switches (no producers, skeleton, ...) + role clocks
mkdir -p gpurun_out/q
for r in 1 2; do
  SPK_PREC=auto timeout 300 python scripts/time_conv.py c2 base >> gpurun_out/q/conv.txt 2>&1
  for v in e32768 e32928 e168 e2048; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python scripts/time_conv.py c2 $v >> gpurun_out/q/conv.txt 2>&1 || echo "$v fail" >> gpurun_out/q/conv.txt; done
done
SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_prof.so timeout 300 python scripts/prof_conv.py c2 > gpurun_out/q/prof.txt 2>&1
