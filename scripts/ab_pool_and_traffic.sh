# A/B of the pooling dispatch threshold (SPK_POOL_SMEM_MIN) on C2, plus pool parity with the smem path forced.
O=gpurun_out; mkdir -p $O
SPK_POOL_SMEM_MIN=0 timeout 600 python -m pytest tests -m gpu -q -k "pool" > $O/pool_tests_smem.log 2>&1; echo "rc=$?" >> $O/pool_tests_smem.log
for v in 2048 0 2048 0; do
  SPK_POOL_SMEM_MIN=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > $O/ab_pool_$v.json 2>> $O/ab_pool.err
  python -c "import json; d=json.load(open('$O/ab_pool_$v.json')); print('$v', d['value'], d['stage_ms']['pool1'])" >> $O/ab_pool.txt
done
bash scripts/ncu_traffic_all.sh
