# A/B: 16 epilogue warps (4 per TMEM lane quadrant, one 16-column chunk each; 28 warps, 72 registers) vs 8
mkdir -p gpurun_out/aa
for r in 1 2; do for c in c2 c4; do for v in ep8 ep16; do
  SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py $c $v >> gpurun_out/aa/conv.txt 2>&1 || echo "$v fail" >> gpurun_out/aa/conv.txt
done; done; done
SPK_LIB_OVERRIDE=exp/libspk_ep16.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or pipeline or full_batch or digit or rate" > gpurun_out/aa/tests.log 2>&1; echo rc=$? >> gpurun_out/aa/tests.log
