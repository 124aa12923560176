# role clocks (epilogue split) of the T = 1 tcgen05 path on C6 (64 images = 19,200 one-step samples)
mkdir -p gpurun_out/jj
SPK_LIB_OVERRIDE=exp/libspk_prof.so timeout 300 python scripts/prof_rate.py 64 > gpurun_out/jj/prof_c6.txt 2>&1
