# One ncu --set full capture of every conv launch of C1, C4 and C5 (one launch per layer,
# scripts/conv_once.py) for the roofline `traffic` field; C2's comes from round_artifacts.sh.
O=gpurun_out; mkdir -p $O
for c in c1 c4 c5; do
  SPK_PREC=auto timeout 900 ncu --set full -k regex:"conv_(tc|event)_kernel" -c 3 -f -o $O/${c}_convs \
      python scripts/conv_once.py $c > $O/ncu_full_$c.log 2>&1
  echo "$c rc=$?" >> $O/ncu_full_$c.log
done
ls -la $O
