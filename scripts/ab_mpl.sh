# event conv: one vs two output maps per lane (SPK_EV_MPL), all layers on the event form where supported
mkdir -p gpurun_out; rm -f gpurun_out/mpl.txt
for c in c2 c4 c5; do for m in 2 4 0; do
  SPK_EV_MPL=$m SPK_PREC=event timeout 300 python scripts/time_conv.py $c mpl$m-$c >> gpurun_out/mpl.txt 2>&1 || echo "$c $m fail" >> gpurun_out/mpl.txt
done; done
