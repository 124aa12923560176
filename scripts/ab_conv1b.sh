mkdir -p gpurun_out; rm -f gpurun_out/ab_conv1b.txt
for c in c2 c4; do
SPK_PREC=auto timeout 120 python scripts/time_conv.py $c base >> gpurun_out/ab_conv1b.txt 2>&1
for v in idle0 epw both test all3; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 90 python scripts/time_conv.py $c $v >> gpurun_out/ab_conv1b.txt 2>&1 || echo "$v fail" >> gpurun_out/ab_conv1b.txt; done
done
