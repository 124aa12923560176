# N-tile / accumulator-buffer sweep on the large configs (C4, C5): does NB=2 with smaller N tiles beat NB=1?
mkdir -p gpurun_out/t
for c in c5 c4; do
  for nt in 0 32 48 64 80 96; do
    SPK_CONV_NT=$nt SPK_PREC=auto timeout 300 python scripts/time_conv.py $c nt$nt >> gpurun_out/t/sweep.txt 2>&1 || echo "$c nt$nt fail" >> gpurun_out/t/sweep.txt
  done
  echo "-- $c" >> gpurun_out/t/sweep.txt
done
