# A/B: conv_tc setup before the PDL wait (in-tree) vs wait at kernel start (tchead); conv / pipeline tests
mkdir -p gpurun_out/rr
for r in 1 2 3; do for v in in tchead; do for c in c2 c4; do
  if [ $v = in ]; then timeout 200 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/rr/b.json 2>/dev/null
  else SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 200 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/rr/b.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/rr/b.json').read().strip().splitlines()[-1]); print('$v $c', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stage_ms'].items() if k.startswith('conv')})" >> gpurun_out/rr/ab.txt
done; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or pipeline or full_batch or digit or rate or fc or host_io" > gpurun_out/rr/tests.log 2>&1; echo rc=$? >> gpurun_out/rr/tests.log
