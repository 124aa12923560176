# A/B of the unrolled fixed-window pooling kernel (SPK_POOL_FIXED) on C2, plus the GPU tests.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
for v in 1 0 1 0; do
  SPK_POOL_FIXED=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > $O/ab_fixed_$v.json 2>> $O/ab_fixed.err
  python -c "import json; d=json.load(open('$O/ab_fixed_$v.json')); print('$v', d['value'], d['stage_ms']['pool1'])" >> $O/ab_fixed.txt
done
