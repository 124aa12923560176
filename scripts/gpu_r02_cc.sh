# role clocks of the tcgen05 conv with the epilogue split into wait / bar.sync / work / tail (C2, C4)
mkdir -p gpurun_out/cc
SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_prof.so timeout 300 python scripts/prof_conv.py c2 > gpurun_out/cc/prof_c2.txt 2>&1
SPK_PREC=auto SPK_LIB_OVERRIDE=exp/libspk_prof.so timeout 300 python scripts/prof_conv.py c4 > gpurun_out/cc/prof_c4.txt 2>&1
