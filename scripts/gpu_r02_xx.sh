# FC and ZCA e2e through one host I/O graph
mkdir -p gpurun_out/xx
for c in fc zca; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/xx/bench_$c.json 2> gpurun_out/xx/bench_$c.err; done
