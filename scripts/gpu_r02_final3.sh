# round 2 closing run on the final tree: GPU suite + parity report, smoke, C2/C3/C2q/C4 bench lines, launch list
mkdir -p gpurun_out/final3
export SPK_PARITY_REPORT=gpurun_out/final3/parity_report.json
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final3/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/final3/gpu_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3/smoke.log 2>&1; echo rc=$? >> gpurun_out/final3/smoke.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final3/gpu.txt
timeout 400 python bench.py > gpurun_out/final3/bench_c2.json 2> gpurun_out/final3/bench_c2.err
for c in c3 c2q c4 c1 c6; do timeout 300 python bench.py --config $c > gpurun_out/final3/bench_$c.json 2> gpurun_out/final3/bench_$c.err; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final3/plain_for_ncu.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final3/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final3/ncu_launches.log 2>&1
