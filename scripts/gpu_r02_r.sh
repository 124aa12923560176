# A/B: mbarrier try_wait suspend-time hints in the tcgen05 conv; streaming gather/pool kernels
mkdir -p gpurun_out/r
for c in c2 c4; do for r in 1 2; do
  SPK_PREC=auto timeout 300 python scripts/time_conv.py $c base >> gpurun_out/r/conv.txt 2>&1
  for v in h1k h20k h1ka h20ka; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 200 python scripts/time_conv.py $c $v >> gpurun_out/r/conv.txt 2>&1 || echo "$v fail" >> gpurun_out/r/conv.txt; done
done; echo "-- $c" >> gpurun_out/r/conv.txt; done
timeout 600 python scripts/bw_kernels.py > gpurun_out/r/bw_base.jsonl 2> gpurun_out/r/bw_base.err
SPK_LIB_OVERRIDE=exp/libspk_bw.so timeout 600 python scripts/bw_kernels.py > gpurun_out/r/bw_new.jsonl 2> gpurun_out/r/bw_new.err
SPK_LIB_OVERRIDE=exp/libspk_bw.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pool or gather" > gpurun_out/r/tests_bw.log 2>&1; echo rc=$? >> gpurun_out/r/tests_bw.log
