# round 2 call d: compute-sanitizer memcheck over every kernel family + conv1 N-tile sweep
mkdir -p gpurun_out
timeout 120 python scripts/sanitize_once.py > gpurun_out/d_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python scripts/sanitize_once.py > gpurun_out/d_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/d_memcheck.log
rm -f gpurun_out/d_sweep.txt
for cfg in "0 2" "128 1" "96 1" "112 1"; do set -- $cfg
  SPK_CONV_NT=$1 SPK_CONV_NB=$2 SPK_PREC=auto timeout 90 python scripts/time_conv.py c2 nt$1-nb$2 >> gpurun_out/d_sweep.txt 2>&1
done
