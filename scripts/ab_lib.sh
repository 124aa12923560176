# C2 bench stage times for libspk variants: ab_lib.sh base VARIANT...
mkdir -p gpurun_out; rm -f gpurun_out/lib_ab.txt
for v in "$@"; do
  if [ $v = base ]; then timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b_$v.json 2>/dev/null
  else SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b_$v.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/b_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), {k: round(x, 4) for k, x in d['stage_ms'].items()})" >> gpurun_out/lib_ab.txt
done
