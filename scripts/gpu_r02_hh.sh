# A/B: STDP kernel before (sthead) and after (stnew) the tile-width heuristic, C2 and C3 bench stage times
mkdir -p gpurun_out/hh
for r in 1 2 3; do for v in sthead stnew; do for c in c2 c3; do
  SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/hh/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/hh/b.json').read().strip().splitlines()[-1]); print('$v $c', round(d['stage_ms']['stdp'],4), round(d['ms_per_step'],4))" >> gpurun_out/hh/ab.txt
done; done; done
