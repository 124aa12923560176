mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on -k regex:rank_code_hist -s 1 -c 1 -f -o gpurun_out/rank_c5 python scripts/prof_stage.py c5 rank_code 592 > gpurun_out/ncu_rank.log 2>&1
timeout 300 ncu --set full --import-source on -k regex:wta_cluster -s 1 -c 1 -f -o gpurun_out/wta_c4 python scripts/prof_stage.py c4 wta > gpurun_out/ncu_wta.log 2>&1
timeout 300 ncu --set full --import-source on -k regex:inhibit_wide -s 1 -c 1 -f -o gpurun_out/inh_c4 python scripts/prof_stage.py c4 inhibit > gpurun_out/ncu_inh.log 2>&1
