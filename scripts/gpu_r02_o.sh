# A/B: trimmed weight stream (in-tree build) vs HEAD (exp/libspk_base.so); rank-code run aggregation
mkdir -p gpurun_out/o
for c in c2 c2q c4 c6 c5; do for r in 1 2; do
  SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_base.so timeout 300 python scripts/time_conv.py $c base >> gpurun_out/o/conv.txt 2>&1
  SPK_PREC=auto timeout 300 python scripts/time_conv.py $c trim >> gpurun_out/o/conv.txt 2>&1
done; echo "-- $c" >> gpurun_out/o/conv.txt; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or pipeline or full_batch or digit or rate or fc" > gpurun_out/o/tests.log 2>&1; echo rc=$? >> gpurun_out/o/tests.log
cp scripts/ab_lib.sh /tmp/ab_lib.sh; cd $GRAFT_REPO_ROOT
for v in base runs base runs; do
  SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/o/b_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/o/b_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), {k: round(x, 4) for k, x in d['stage_ms'].items()})" >> gpurun_out/o/lib_ab.txt
done
