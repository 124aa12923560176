# round 2 call e: full GPU suite, smoke, benches (fused inhibit+WTA, per-device attrs, STDP status)
mkdir -p gpurun_out
export SPK_PARITY_REPORT=gpurun_out/parity_report_r02e.json
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/e_tests.log 2>&1; echo rc=$? >> gpurun_out/e_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1
for c in c2 c3 c4 c1; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/e_bench_$c.json 2> gpurun_out/e_bench_$c.err; done
