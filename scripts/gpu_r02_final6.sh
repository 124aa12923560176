# round 2 closing evidence run v6 (PDL launch chain, vectorized weight pack, STDP forms, host I/O graph): GPU suite, smoke, every bench line, reference arm, launch list, ncu of the C2 convs
# ncu launch list of the headline bench, ncu --set full of the C2 tcgen05 convs
mkdir -p gpurun_out/final6
export SPK_PARITY_REPORT=gpurun_out/final6/parity_report.json
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final6/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/final6/gpu_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6/smoke.log 2>&1; echo rc=$? >> gpurun_out/final6/smoke.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final6/gpu.txt
timeout 400 python bench.py > gpurun_out/final6/bench_c2.json 2> gpurun_out/final6/bench_c2.err
for c in c1 c3 c4 c2q c6 fc zca; do timeout 300 python bench.py --config $c > gpurun_out/final6/bench_$c.json 2> gpurun_out/final6/bench_$c.err; done
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/final6/bench_c5.json 2> gpurun_out/final6/bench_c5.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final6/reference_c2.json 2> gpurun_out/final6/reference_c2.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final6/plain_for_ncu.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final6/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final6/ncu_launches.log 2>&1
SPK_PREC=auto timeout 300 python scripts/conv_once.py c2 > gpurun_out/final6/conv_once.log 2>&1 && \
SPK_PREC=auto timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -c 2 -o gpurun_out/final6/conv_c2 python scripts/conv_once.py c2 > gpurun_out/final6/ncu_full.log 2>&1
