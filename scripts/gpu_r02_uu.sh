# packed-weight kernel with 4 synapses per thread: conv / digit-plane / pipeline tests, C2 bench x3, launch list
mkdir -p gpurun_out/uu
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or digit or pipeline or full_batch or fc or rate or clamp" > gpurun_out/uu/tests.log 2>&1; echo rc=$? >> gpurun_out/uu/tests.log
for r in 1 2 3; do timeout 200 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/uu/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/uu/b.json').read().strip().splitlines()[-1]); print('c2', round(d['ms_per_step'],4), round(d['stage_ms']['conv2'],4))" >> gpurun_out/uu/ab.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pack_weights -c 5 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/uu/ncu_pack.csv 2>&1
