# STDP tile-width heuristic in-tree: STDP / pipeline / FC parity tests and C2, C3 bench lines
mkdir -p gpurun_out/gg
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "stdp or pipeline or full_batch or fc or smoke" > gpurun_out/gg/tests.log 2>&1; echo rc=$? >> gpurun_out/gg/tests.log
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/gg/bench_$c.json 2>/dev/null; done
