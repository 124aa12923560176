# A/B: STDP update weights per CTA (kUpdW 32 in-tree vs 64 / 128): C2 and C3 bench stage times; STDP parity tests
mkdir -p gpurun_out/ff
for r in 1 2; do for v in in st64 st128; do for c in c2 c3; do
  if [ $v = in ]; then timeout 120 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/ff/b.json 2>/dev/null
  else SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/ff/b.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/ff/b.json').read().strip().splitlines()[-1]); print('$v $c', round(d['stage_ms']['stdp'],4), round(d['ms_per_step'],4))" >> gpurun_out/ff/stdp_ab.txt
done; done; done
for v in st64 st128; do SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stdp or pipeline or full_batch" > gpurun_out/ff/tests_$v.log 2>&1; echo "$v rc=$?" >> gpurun_out/ff/tests.txt; done
