# A/B: P* crossing by lowest set bit for TP = 32 (in-tree) vs HEAD (exp/libspk_head.so), auto engines, C4 and C2
mkdir -p gpurun_out/zz
for r in 1 2 3; do for c in c4 c2; do
  SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_head.so timeout 300 python scripts/time_conv.py $c head >> gpurun_out/zz/conv.txt 2>&1
  SPK_PREC=auto timeout 300 python scripts/time_conv.py $c new >> gpurun_out/zz/conv.txt 2>&1
done; done
