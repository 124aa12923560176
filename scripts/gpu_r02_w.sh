# A/B: rank coding cluster kernel with peer groups copied locally (rcs2, rcs4) vs one CTA per sample (rcs0)
mkdir -p gpurun_out/w
for v in rcs0 rcs2 rcs4 rcs2; do
  SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/bw_kernels.py --quick > gpurun_out/w/bw_$v.jsonl 2>/dev/null
  grep rank_code gpurun_out/w/bw_$v.jsonl | sed "s/^/$v /" >> gpurun_out/w/rank_ab.txt
done
SPK_LIB_OVERRIDE=exp/libspk_rcs2.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rank" > gpurun_out/w/tests_rcs2.log 2>&1; echo rc=$? >> gpurun_out/w/tests_rcs2.log
