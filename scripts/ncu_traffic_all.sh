# One ncu --set full capture of every conv launch of C1 and C4 (one launch per layer,
# scripts/conv_once.py) for the roofline `traffic` field; C2's comes from round_artifacts.sh.
# The DRAM bytes are extracted on the box (the reports exceed gpurun's copy-back limit).
O=gpurun_out; mkdir -p $O
cp profiles/ncu_traffic.json $O/ncu_traffic.json
for c in c1 c4; do
  SPK_PREC=auto timeout 600 ncu --set full -k regex:"conv_(tc|event)_kernel" -c 3 -f -o $O/${c}_convs \
      python scripts/conv_once.py $c > $O/ncu_full_$c.log 2>&1
  echo "$c rc=$?" >> $O/ncu_full_$c.log
  TRAFFIC_OUT=$O/ncu_traffic.json python scripts/ncu_traffic_update.py $c >> $O/ncu_full_$c.log 2>&1
  ncu -i $O/${c}_convs.ncu-rep --page details --csv > $O/${c}_convs_details.csv 2>/dev/null
  rm -f $O/${c}_convs.ncu-rep
done
ls -la $O
