# Round-end evidence on one B200: GPU tests, smoke, bench lines (C1-C5, reference arm, --dp),
# the ncu launch list of the C2 bench command and one ncu --set full capture per C2 conv layer.
set -x
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_c2.json 2> $O/reference_c2.err
for c in c1 c3 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 3 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 300 python bench.py --dp --no-cpu-baseline > $O/bench_c2_dp.json 2> $O/bench_c2_dp.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
SPK_PREC=auto timeout 600 ncu --set full --import-source on -k regex:"conv_(tc|event)_kernel" -c 3 -f -o $O/c2_convs python scripts/conv_once.py c2 > $O/ncu_full.log 2>&1
ls -la $O
