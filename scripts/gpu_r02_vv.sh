# A/B: per-weight fused STDP update (SPK_STDP_PW=1, default) vs two-phase tiles; STDP / pipeline / FC tests
mkdir -p gpurun_out/vv
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "stdp or pipeline or full_batch or fc or smoke or data_parallel or host_io or run_twice" > gpurun_out/vv/tests.log 2>&1; echo rc=$? >> gpurun_out/vv/tests.log
for r in 1 2 3; do for v in 1 0; do for c in c2 c3 c1 fc; do
  SPK_STDP_PW=$v timeout 200 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/vv/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/vv/b.json').read().strip().splitlines()[-1]); print('pw=$v $c', round(d['ms_per_step'],4), round(d['stage_ms'].get('stdp', 0),4))" >> gpurun_out/vv/ab.txt
done; done; done
