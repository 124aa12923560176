# tcgen05 conv plan knobs on C2 (conv1, conv2) and C4 (conv1): SPK_CONV_RETAIN x SPK_CONV_NT x SPK_CONV_G
mkdir -p gpurun_out; rm -f gpurun_out/sweep.txt
for r in 1 0; do for nt in 0 128 96 80; do for g in 2 1; do
  SPK_CONV_RETAIN=$r SPK_CONV_NT=$nt SPK_CONV_G=$g SPK_PREC=auto timeout 60 python scripts/time_conv.py c2 r$r-nt$nt-g$g >> gpurun_out/sweep.txt 2>&1 || echo "c2 r$r nt$nt g$g fail" >> gpurun_out/sweep.txt
done; done; done
