mkdir -p gpurun_out
SPK_BENCH_TRACE=1 timeout 100 python -X faulthandler bench.py --config zca --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/i_zca.json 2> gpurun_out/i_zca.err; echo rc=$? >> gpurun_out/i_zca.err
SPK_BENCH_TRACE=1 timeout 100 python -X faulthandler bench.py --config fc --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/i_fc.json 2> gpurun_out/i_fc.err; echo rc=$? >> gpurun_out/i_fc.err
timeout 300 python -m pytest tests/test_gpu_next.py -q -x -k "rate" > gpurun_out/i_tests.log 2>&1; echo rc=$? >> gpurun_out/i_tests.log
timeout 300 python bench.py --config c6 --no-cpu-baseline > gpurun_out/i_bench_c6.json 2> gpurun_out/i_bench_c6.err
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/i_bench_c2.json 2> gpurun_out/i_bench_c2.err
