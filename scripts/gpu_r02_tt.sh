# full GPU suite + smoke + C2/C1 bench on the in-tree build (conv_tc setup before the PDL wait)
mkdir -p gpurun_out/tt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tt/tests.log 2>&1; echo rc=$? >> gpurun_out/tt/tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/tt/smoke.log 2>&1; echo rc=$? >> gpurun_out/tt/smoke.log
for c in c2 c1 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/tt/bench_$c.json 2> gpurun_out/tt/bench_$c.err; done
