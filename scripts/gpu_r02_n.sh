mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_next.py tests/test_gpu_parity.py -q -x -k "fire or fc or rate" > gpurun_out/n_tests.log 2>&1; echo rc=$? >> gpurun_out/n_tests.log
timeout 600 python scripts/bw_kernels.py > gpurun_out/n_bw.jsonl 2> gpurun_out/n_bw.err
timeout 300 python bench.py --config c6 --no-cpu-baseline > gpurun_out/n_bench_c6.json 2> gpurun_out/n_bench_c6.err
