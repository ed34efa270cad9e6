set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r2_pytest_gpu6.txt 2>&1; tail -5 gpurun_out/r2_pytest_gpu6.txt
timeout 300 python tools/mc_cta_replay.py cfg2 > gpurun_out/r2_mc_cta_cfg2_v4.txt 2>&1; tail -2 gpurun_out/r2_mc_cta_cfg2_v4.txt
MSG_HOST_PHASES=1 timeout 300 python tools/prof_replay.py cfg2 3 > gpurun_out/r2_host_phases_cfg2.txt 2>&1; cat gpurun_out/r2_host_phases_cfg2.txt
timeout 600 python tools/prof_replay.py frag 2 > gpurun_out/r2_frag_replay_v4.txt 2>&1; cat gpurun_out/r2_frag_replay_v4.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_frag_v4.csv python tools/prof_replay.py frag 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_launches_frag_v4.csv > gpurun_out/r2_launches_frag_v4_summary.txt 2>&1; head -12 gpurun_out/r2_launches_frag_v4_summary.txt
