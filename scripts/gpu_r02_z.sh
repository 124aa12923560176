# A/B: event conv counting sort with one shared atomic per equal-latency group (evm) vs per lane (ev0)
mkdir -p gpurun_out/z
for r in 1 2; do for c in c2 c4 c1; do for v in ev0 evm; do
  SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py $c $v >> gpurun_out/z/conv.txt 2>&1
done; done; done
for v in ev0 evm; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py c5 $v >> gpurun_out/z/conv.txt 2>&1; done
SPK_LIB_OVERRIDE=exp/libspk_evm.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or event or pipeline or rate or fc" > gpurun_out/z/tests.log 2>&1; echo rc=$? >> gpurun_out/z/tests.log
