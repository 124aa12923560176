# A/B of conv_tc timing-experiment variants (exp/libspk_*.so) on C2 and C4 (SPK_PREC=auto); each run bounded
mkdir -p gpurun_out; rm -f gpurun_out/ab_tc.txt
for c in c2 c4; do
  SPK_PREC=auto timeout 120 python scripts/time_conv.py $c base >> gpurun_out/ab_tc.txt 2>&1
  for v in "$@"; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 60 python scripts/time_conv.py $c $v >> gpurun_out/ab_tc.txt 2>&1 || echo "$c $v timeout/fail" >> gpurun_out/ab_tc.txt; done
done
