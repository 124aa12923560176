# rerun of the tchead arm of gpu_r02_rr.sh with errors kept
mkdir -p gpurun_out/ss
for r in 1 2 3; do for v in tchead in; do
  if [ $v = in ]; then timeout 200 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ss/b_$v.json 2> gpurun_out/ss/b_$v.err
  else SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 200 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ss/b_$v.json 2> gpurun_out/ss/b_$v.err; fi
  python -c "import json; d=json.loads(open('gpurun_out/ss/b_$v.json').read().strip().splitlines()[-1]); print('$v c2', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stage_ms'].items() if k.startswith('conv')})" >> gpurun_out/ss/ab.txt 2>> gpurun_out/ss/py.err
done; done
