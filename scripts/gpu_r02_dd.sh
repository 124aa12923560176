# A/B: fire-epilogue tests / ballots / selection as separate unrolled phases (ilp) vs fused per column (noilp)
mkdir -p gpurun_out/dd
for r in 1 2; do for c in c2 c4; do for v in noilp ilp; do
  SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_$v.so timeout 300 python scripts/time_conv.py $c $v >> gpurun_out/dd/conv.txt 2>&1 || echo "$v fail" >> gpurun_out/dd/conv.txt
done; done; done
