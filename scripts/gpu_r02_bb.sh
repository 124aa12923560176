# A/B: MMA issue by one elected thread as straight-line uniform code (lean: retained-A fast path;
# lean2: every hand-off) vs the per-MMA elect.sync asm blocks (nolean)
mkdir -p gpurun_out/bb
for r in 1 2; do for c in c2 c4; do for v in nolean lean lean2; do
  SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py $c $v >> gpurun_out/bb/conv.txt 2>&1 || echo "$v fail" >> gpurun_out/bb/conv.txt
done; done; done
for v in nolean lean2; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py c5 $v >> gpurun_out/bb/conv.txt 2>&1; done
SPK_LIB_OVERRIDE=exp/libspk_lean2.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or pipeline or full_batch or digit or rate or fc" > gpurun_out/bb/tests.log 2>&1; echo rc=$? >> gpurun_out/bb/tests.log
for v in nolean lean2; do SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bb/bench_$v.json 2>/dev/null; done
