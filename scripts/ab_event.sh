# A/B of the event conv against exp/libspk_old.so + event parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or pipeline or forward" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
rm -f gpurun_out/ab.txt
for c in c2 c4; do
SPK_PREC=event SPK_LIB_OVERRIDE=exp/libspk_old.so python scripts/time_conv.py $c old >> gpurun_out/ab.txt 2>&1
SPK_PREC=event python scripts/time_conv.py $c new >> gpurun_out/ab.txt 2>&1
done
SPK_PREC=event timeout 600 ncu --set full --import-source on -k regex:conv_event -c 1 -f -o gpurun_out/ev_new python scripts/time_conv.py c2 x > /dev/null 2>&1
