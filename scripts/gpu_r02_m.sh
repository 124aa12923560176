mkdir -p gpurun_out
export SPK_PARITY_REPORT=gpurun_out/parity_report_r02m.json
timeout 600 python -m pytest tests/test_gpu_next.py tests/test_gpu_parity.py -q -x -k "fire or fc or rate" > gpurun_out/m_tests.log 2>&1; echo rc=$? >> gpurun_out/m_tests.log
timeout 200 python bench.py --config fc --no-cpu-baseline > gpurun_out/m_fc.json 2> gpurun_out/m_fc.err
timeout 600 python scripts/bw_kernels.py > gpurun_out/m_bw.jsonl 2> gpurun_out/m_bw.err
