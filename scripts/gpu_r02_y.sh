# T = 1 path: kernel rows padded to 8 synapses and read as words (SPK_CONV_ROWPAD=1, default) vs the
# synapse-by-synapse gather (SPK_CONV_ROWPAD=0); GPU tests of the conv engines and the rate pipeline
mkdir -p gpurun_out/y
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or rate or pipeline or fc" > gpurun_out/y/tests.log 2>&1; echo rc=$? >> gpurun_out/y/tests.log
for r in 1 2; do
  for v in 1 0; do
    SPK_CONV_ROWPAD=$v timeout 300 python bench.py --config c6 --no-cpu-baseline > gpurun_out/y/c6_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/y/c6_$v.json').read().strip().splitlines()[-1]); print('rowpad=$v', round(d['ms_per_step'],3), d['value'], {k: round(x,3) for k,x in d['stage_ms'].items()})" >> gpurun_out/y/c6_ab.txt
  done
done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/y/c2.json 2>/dev/null
