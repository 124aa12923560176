# A/B of STDP update tilings (exp/libspk_st*.so) on the C2 bench step
mkdir -p gpurun_out; rm -f gpurun_out/stdp_ab.txt
for v in "$@"; do
  if [ $v = base ]; then timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b_$v.json 2>/dev/null
  else SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b_$v.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/b_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['stage_ms']['stdp'],4), round(d['ms_per_step'],4))" >> gpurun_out/stdp_ab.txt
done
