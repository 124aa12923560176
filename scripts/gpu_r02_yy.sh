# A/B: P* crossing test by lowest set bit for one-pixel warps (TP = 32: C4's trained layer); in-tree = new.
# Baseline = the previous run's numbers (gpu_r02_final6 / bench c4); conv/pipeline tests
mkdir -p gpurun_out/yy
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "conv or pipeline or full_batch or digit" > gpurun_out/yy/tests.log 2>&1; echo rc=$? >> gpurun_out/yy/tests.log
for r in 1 2 3; do timeout 300 python scripts/time_conv.py c4 new >> gpurun_out/yy/conv.txt 2>&1; done
