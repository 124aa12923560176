# quick GPU check: selected parity tests + C2/C4/C5 bench lines (pass pytest -k expr as $1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
