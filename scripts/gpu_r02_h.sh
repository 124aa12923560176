mkdir -p gpurun_out
export SPK_PARITY_REPORT=gpurun_out/parity_report_r02h.json
SPK_BENCH_WATCHDOG=60 timeout 100 python bench.py --config fc --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/h_fc.json 2> gpurun_out/h_fc.err; echo rc=$? >> gpurun_out/h_fc.err
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_parity.py -m gpu -q -x -k "rate or conv_potentials or conv_fire or T1 or quantised" > gpurun_out/h_tests.log 2>&1; echo rc=$? >> gpurun_out/h_tests.log
timeout 300 python bench.py --config c6 --no-cpu-baseline > gpurun_out/h_bench_c6.json 2> gpurun_out/h_bench_c6.err
