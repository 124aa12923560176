# C2 conv plan knobs: N tile x hand-off group x accumulator buffers (time_conv.py prints conv0 conv1 conv2 ms)
mkdir -p gpurun_out; rm -f gpurun_out/sweep_c2.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/sweep_c2.txt
for nt in 0 32 48 64; do for g in 2 1; do for nb in 2 1; do
  SPK_CONV_NT=$nt SPK_CONV_G=$g SPK_CONV_NB=$nb SPK_PREC=auto timeout 90 python scripts/time_conv.py c2 nt$nt-g$g-nb$nb >> gpurun_out/sweep_c2.txt 2>&1 || echo "nt$nt g$g nb$nb fail" >> gpurun_out/sweep_c2.txt
done; done; done
