# A/B: lean single-thread MMA issue on the retained-A fast path (ln1) vs per-MMA elect (ln0): full C2, C3, C4 bench steps
mkdir -p gpurun_out/mm
for r in 1 2 3; do for v in ln0 ln1; do for c in c2 c4; do
  SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 200 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/mm/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/mm/b.json').read().strip().splitlines()[-1]); print('$v $c', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms'].items() if k.startswith('conv')})" >> gpurun_out/mm/ab.txt
done; done; done
SPK_LIB_OVERRIDE=exp/libspk_ln1.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "conv or pipeline or full_batch or digit" > gpurun_out/mm/tests.log 2>&1; echo rc=$? >> gpurun_out/mm/tests.log
