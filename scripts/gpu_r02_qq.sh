# A/B: programmatic dependent launch on every libspk kernel (SPK_PDL=1, default) vs off; full GPU suite with PDL
mkdir -p gpurun_out/qq
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/qq/tests.log 2>&1; echo rc=$? >> gpurun_out/qq/tests.log
for r in 1 2 3; do for v in 1 0; do for c in c2 c1 c4; do
  SPK_PDL=$v timeout 200 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/qq/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/qq/b.json').read().strip().splitlines()[-1]); print('pdl=$v $c', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'value', round(d['value']))" >> gpurun_out/qq/ab.txt
done; done; done
