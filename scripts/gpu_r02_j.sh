mkdir -p gpurun_out
SPK_LIB_OVERRIDE=exp/libspk_prof.so timeout 200 python scripts/prof_rate.py 64 > gpurun_out/j_prof_rate.txt 2>&1
SPK_BENCH_TRACE=1 timeout 200 python bench.py --config fc --no-cpu-baseline > gpurun_out/j_fc.json 2> gpurun_out/j_fc.err
SPK_BENCH_TRACE=1 timeout 200 python bench.py --config zca --no-cpu-baseline > gpurun_out/j_zca.json 2> gpurun_out/j_zca.err
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "inhibit or wta or pipeline" > gpurun_out/j_tests.log 2>&1; echo rc=$? >> gpurun_out/j_tests.log
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/j_bench_c2.json 2> gpurun_out/j_bench_c2.err
