set -x
MSG_HOST_PHASES=1 timeout 300 python tools/prof_replay.py cfg2 3 > gpurun_out/r2_host_phases_cfg2_v2.txt 2>&1; cat gpurun_out/r2_host_phases_cfg2_v2.txt
MSG_HOST_PHASES=1 timeout 300 python tools/prof_replay.py cfg4 2 > gpurun_out/r2_host_phases_cfg4.txt 2>&1; cat gpurun_out/r2_host_phases_cfg4.txt
