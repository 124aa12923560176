mkdir -p gpurun_out; rm -f gpurun_out/r_ab.txt
for c in c2 c2q; do for v in base fast base fast; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python scripts/time_conv.py $c $v >> gpurun_out/r_ab.txt 2>&1; done; done
SPK_LIB_OVERRIDE=exp/libspk_fast.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "conv_potentials or conv_fire_epilogue or pipeline_c2 or live_digit or full_batch" > gpurun_out/r_tests.log 2>&1; echo rc=$? >> gpurun_out/r_tests.log
