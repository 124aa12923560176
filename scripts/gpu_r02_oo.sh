# GPU test of Network.capture_io, plus the determinism / sharded-forward tests around it
mkdir -p gpurun_out/oo
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host_io or run_twice or sharded" > gpurun_out/oo/tests.log 2>&1; echo rc=$? >> gpurun_out/oo/tests.log
