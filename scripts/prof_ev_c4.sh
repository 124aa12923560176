mkdir -p gpurun_out
SPK_PREC=event timeout 600 ncu --set full --import-source on -k regex:conv_event -s 1 -c 1 -f -o gpurun_out/ev_c4l1 python scripts/conv_once.py c4 64 > gpurun_out/ncu_ev.log 2>&1
