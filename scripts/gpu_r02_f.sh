mkdir -p gpurun_out
export SPK_PARITY_REPORT=gpurun_out/parity_report_r02f.json
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f_tests.log 2>&1; echo rc=$? >> gpurun_out/f_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
for c in c2 c4 fc zca; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/f_bench_$c.json 2> gpurun_out/f_bench_$c.err; done
rm -f gpurun_out/f_ab.txt
for c in c2 c4; do for v in base0 pipe; do SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 120 python scripts/time_conv.py $c $v >> gpurun_out/f_ab.txt 2>&1; done; done
