# A/B: fused inhibit+WTA mode 4 (two quads per thread, prefetched latency words); ncu --set full of the C2 event conv
mkdir -p gpurun_out/u
for v in base wta wta2 base wta wta2; do
  if [ $v = base ]; then timeout 300 python scripts/bw_kernels.py > gpurun_out/u/bw_$v.jsonl 2>/dev/null
  else SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/bw_kernels.py > gpurun_out/u/bw_$v.jsonl 2>/dev/null; fi
  grep -h "inhibit_wta\|wta (" gpurun_out/u/bw_$v.jsonl | sed "s/^/$v /" >> gpurun_out/u/wta_ab.txt
done
SPK_LIB_OVERRIDE=exp/libspk_wta.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wta or inhibit or pipeline or full_batch" > gpurun_out/u/tests_wta.log 2>&1; echo rc=$? >> gpurun_out/u/tests_wta.log
SPK_PREC=auto timeout 300 python scripts/conv_once.py c2 > gpurun_out/u/conv_once.log 2>&1 && \
SPK_PREC=auto timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_event_kernel -c 1 -o gpurun_out/u/conv_event_c2 python scripts/conv_once.py c2 > gpurun_out/u/ncu.log 2>&1
