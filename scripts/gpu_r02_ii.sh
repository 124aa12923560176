# A/B: threads per CTA of the 32-weight STDP update tile (C2 layer 3): 256 / 128 / 64; STDP tests on the winner
mkdir -p gpurun_out/ii
for r in 1 2 3; do for v in t256 t128 t64; do
  SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ii/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ii/b.json').read().strip().splitlines()[-1]); print('$v', round(d['stage_ms']['stdp'],4), round(d['ms_per_step'],4))" >> gpurun_out/ii/ab.txt
done; done
for v in t128 t64; do SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stdp or full_batch" > gpurun_out/ii/tests_$v.log 2>&1; echo "$v rc=$?" >> gpurun_out/ii/tests.txt; done
