# STDP form selection (per-weight for few winners on short rows): C2/C3/C1/FC bench; STDP tests with the per-weight form forced
mkdir -p gpurun_out/ww
SPK_STDP_PW=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "stdp or pipeline or full_batch or fc or data_parallel or run_twice" > gpurun_out/ww/tests_pw2.log 2>&1; echo rc=$? >> gpurun_out/ww/tests_pw2.log
for r in 1 2; do for c in c2 c3 c1 fc; do
  timeout 200 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/ww/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ww/b.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), round(d['stage_ms'].get('stdp', 0),4), round(d['value']))" >> gpurun_out/ww/ab.txt
done; done
