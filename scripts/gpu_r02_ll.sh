# A/B: 3x3/3 pooling of small planes with one thread per output row (default) vs per output (SPK_POOL_ROW=0); pool tests
mkdir -p gpurun_out/ll
for r in 1 2 3; do for v in 1 0; do
  SPK_POOL_ROW=$v timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ll/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ll/b.json').read().strip().splitlines()[-1]); print('row=$v', round(d['stage_ms']['pool1'],4), round(d['ms_per_step'],4))" >> gpurun_out/ll/ab.txt
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pool or pipeline or full_batch" > gpurun_out/ll/tests.log 2>&1; echo rc=$? >> gpurun_out/ll/tests.log
