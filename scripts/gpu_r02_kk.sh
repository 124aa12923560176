# A/B: fused inhibit+WTA small-slice mode with four channels' loads per trip (wnew) vs one (wold): C1, C2, C3 stage times; WTA tests
mkdir -p gpurun_out/kk
for r in 1 2 3; do for v in wold wnew; do for c in c1 c2; do
  SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/kk/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/kk/b.json').read().strip().splitlines()[-1]); print('$v $c', round(d['stage_ms']['inhibit_wta'],4), round(d['ms_per_step'],4))" >> gpurun_out/kk/ab.txt
done; done; done
SPK_LIB_OVERRIDE=exp/libspk_wnew.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "wta or inhibit or pipeline or full_batch or smoke" > gpurun_out/kk/tests.log 2>&1; echo rc=$? >> gpurun_out/kk/tests.log
