# A/B: DoG filter on small maps (C1-C3) with the 4-rows-per-thread kernel (SPK_FILTER_RB_SMALL=1) vs the 1-row one
mkdir -p gpurun_out/pp
for r in 1 2 3; do for v in 0 1; do for c in c2 c1; do
  SPK_FILTER_RB_SMALL=$v timeout 120 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/pp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pp/b.json').read().strip().splitlines()[-1]); print('rb=$v $c', round(d['stage_ms']['filter'],4), round(d['ms_per_step'],4))" >> gpurun_out/pp/ab.txt
done; done; done
SPK_FILTER_RB_SMALL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "filter or dog or log or gabor or pipeline" > gpurun_out/pp/tests.log 2>&1; echo rc=$? >> gpurun_out/pp/tests.log
