mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_next.py tests/test_gpu_parity.py -q -x -k "rate or conv_potentials or conv_fire_epilogue" > gpurun_out/k_tests.log 2>&1; echo rc=$? >> gpurun_out/k_tests.log
SPK_LIB_OVERRIDE=exp/libspk_prof.so timeout 200 python scripts/prof_rate.py 64 > gpurun_out/k_prof_rate.txt 2>&1
timeout 300 python bench.py --config c6 --no-cpu-baseline > gpurun_out/k_bench_c6.json 2> gpurun_out/k_bench_c6.err
