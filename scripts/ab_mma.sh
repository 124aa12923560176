mkdir -p gpurun_out; rm -f gpurun_out/q_ab.txt
for c in c2 c2q; do for v in base one base one; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python scripts/time_conv.py $c $v >> gpurun_out/q_ab.txt 2>&1; done; done
SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_base.so timeout 120 python scripts/time_conv.py c4 base >> gpurun_out/q_ab.txt 2>&1
SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_one.so timeout 120 python scripts/time_conv.py c4 one >> gpurun_out/q_ab.txt 2>&1
