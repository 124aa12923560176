mkdir -p gpurun_out; rm -f gpurun_out/nt.txt
for nt in 0 64 48 32; do for nb in 2 1; do
 SPK_CONV_NT=$nt SPK_CONV_NB=$nb SPK_PREC=auto timeout 120 python scripts/time_conv.py c4 nt$nt-nb$nb >> gpurun_out/nt.txt 2>&1
 SPK_CONV_NT=$nt SPK_CONV_NB=$nb SPK_PREC=auto timeout 120 python scripts/time_conv.py c2 nt$nt-nb$nb >> gpurun_out/nt.txt 2>&1
done; done
