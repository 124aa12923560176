# e2e through one graph holding the host copies and the step (Network.capture_io): bench lines C2, C3, C4, C6, C1
mkdir -p gpurun_out/nn
for c in c2 c3 c4 c6 c1; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/nn/bench_$c.json 2> gpurun_out/nn/bench_$c.err; done
