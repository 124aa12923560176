mkdir -p gpurun_out
timeout 600 python scripts/bw_kernels.py > gpurun_out/l_bw.jsonl 2> gpurun_out/l_bw.err
timeout 300 python scripts/bw_kernels.py --quick > gpurun_out/l_bw_quick.jsonl 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/l_bw_ncu.csv python scripts/bw_kernels.py --quick > gpurun_out/l_bw_ncu.log 2>&1
