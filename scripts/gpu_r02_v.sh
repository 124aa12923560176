# A/B: rank coding on a cluster of CTAs per sample (in-tree CS=2, rcs4, rcs0 = one CTA per sample);
# event conv ballot walk (in-tree) vs counting sort (evsort); GPU tests of both; C2/C4 bench
mkdir -p gpurun_out/v
for r in 1 2; do
  for c in c2 c1 c4; do
    SPK_PREC=auto timeout 300 python scripts/time_conv.py $c walk >> gpurun_out/v/conv.txt 2>&1
    SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_evsort.so timeout 300 python scripts/time_conv.py $c sort >> gpurun_out/v/conv.txt 2>&1
  done
done
for v in in rcs0 rcs4; do
  if [ $v = in ]; then timeout 300 python scripts/bw_kernels.py > gpurun_out/v/bw_$v.jsonl 2>gpurun_out/v/bw_$v.err
  else SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/bw_kernels.py > gpurun_out/v/bw_$v.jsonl 2>/dev/null; fi
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "rank or conv or pipeline or full_batch or event or rate or fc or smoke" > gpurun_out/v/tests.log 2>&1; echo rc=$? >> gpurun_out/v/tests.log
SPK_LIB_OVERRIDE=exp/libspk_rcs4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rank" > gpurun_out/v/tests_rcs4.log 2>&1; echo rc=$? >> gpurun_out/v/tests_rcs4.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v/bench_c2.json 2> gpurun_out/v/bench_c2.err
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/v/bench_c4.json 2> gpurun_out/v/bench_c4.err
