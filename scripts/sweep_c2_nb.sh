# C2 conv plan knobs round 2: more accumulator buffers (NB up to 4) with narrower N tiles; retain on/off
mkdir -p gpurun_out; rm -f gpurun_out/sweep_nb.txt
for r in 1 0; do for cfg in "0 2" "32 4" "32 3" "16 4" "48 2" "64 2"; do set -- $cfg
  SPK_CONV_RETAIN=$r SPK_CONV_NT=$1 SPK_CONV_NB=$2 SPK_PREC=auto timeout 90 python scripts/time_conv.py c2 r$r-nt$1-nb$2 >> gpurun_out/sweep_nb.txt 2>&1 || echo "r$r nt$1 nb$2 fail" >> gpurun_out/sweep_nb.txt
done; done
for cfg in "0 2" "32 4" "16 4"; do set -- $cfg
  SPK_CONV_NT=$1 SPK_CONV_NB=$2 SPK_PREC=auto timeout 90 python scripts/time_conv.py c2q q-nt$1-nb$2 >> gpurun_out/sweep_nb.txt 2>&1
done
