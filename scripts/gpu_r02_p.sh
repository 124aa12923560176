# A/B: flusher widest-aligned stores (in-tree) vs HEAD (exp/libspk_base.so) vs no flusher stores (e8, timing only)
mkdir -p gpurun_out/p
for c in c2 c4 c2q; do for r in 1 2; do
  for v in base e8; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py $c $v >> gpurun_out/p/conv.txt 2>&1; done
  SPK_PREC=auto timeout 300 python scripts/time_conv.py $c fl >> gpurun_out/p/conv.txt 2>&1
done; echo "-- $c" >> gpurun_out/p/conv.txt; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or pipeline or full_batch or digit" > gpurun_out/p/tests.log 2>&1; echo rc=$? >> gpurun_out/p/tests.log
