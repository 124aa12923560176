# A/B: small-sample rank coding (C2/C3 front end): bucket count and CTA size; the bitonic kernel (SPK_RANK_SORT=1)
mkdir -p gpurun_out/x
for r in 1 2; do
  for v in in sort s20t256 s19t512 s20t512 s19t128; do
    if [ $v = in ]; then timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/x/b_$v.json 2>/dev/null
    elif [ $v = sort ]; then SPK_RANK_SORT=1 timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/x/b_$v.json 2>/dev/null
    else SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/x/b_$v.json 2>/dev/null; fi
    python -c "import json; d=json.loads(open('gpurun_out/x/b_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['stage_ms']['rank_code'],4))" >> gpurun_out/x/rank_small.txt
  done
done
for v in s20t256 s19t512 s20t512 s19t128; do
  SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "rank" > gpurun_out/x/tests_$v.log 2>&1; echo "$v rc=$?" >> gpurun_out/x/tests.txt
done
# ncu --set full of the C6 conv0 launch (TP = 1 path)
timeout 300 python scripts/conv_once_rate.py 64 > gpurun_out/x/conv_once_rate.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -c 1 -o gpurun_out/x/conv_c6 python scripts/conv_once_rate.py 64 > gpurun_out/x/ncu.log 2>&1
