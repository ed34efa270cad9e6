timeout 600 ncu --set full --import-source on --clock-control none -f -k regex:k_ms_coop -s 40 -c 1 -o gpurun_out/r2_ncu_k_ms_coop_cfg2 python tools/prof_replay.py cfg2 1 > /dev/null 2>&1
timeout 300 python tools/mc_cta_replay.py cfg2 > gpurun_out/r2_mc_cta_cfg2_v6.txt 2>&1; tail -2 gpurun_out/r2_mc_cta_cfg2_v6.txt
