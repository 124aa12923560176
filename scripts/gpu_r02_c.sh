# round 2 call c: conv tests, benches of every workload, ncu source capture of C2 conv1
mkdir -p gpurun_out
export SPK_PARITY_REPORT=gpurun_out/parity_report_r02c.json
timeout 900 python -m pytest tests -m gpu -q -x -k "conv or pipeline or full_batch or digit" > gpurun_out/c_tests.log 2>&1; echo rc=$? >> gpurun_out/c_tests.log
for c in c2 c2q c6 c1 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/c_bench_$c.json 2> gpurun_out/c_bench_$c.err; done
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/c_bench_c4.json 2> gpurun_out/c_bench_c4.err
timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/c_bench_c5.json 2> gpurun_out/c_bench_c5.err
SPK_PREC=auto timeout 300 python scripts/conv_once.py c2 > gpurun_out/c_plain.log 2>&1 && \
SPK_PREC=auto timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -c 2 -o gpurun_out/c_conv_c2 python scripts/conv_once.py c2 > gpurun_out/c_ncu.log 2>&1
