set -x
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2_pytest_gpu9.txt 2>&1; tail -5 gpurun_out/r2_pytest_gpu9.txt; grep -E "^FAILED" gpurun_out/r2_pytest_gpu9.txt | head -20
MSG_HOST_PHASES=1 timeout 300 python tools/prof_replay.py cfg2 3 > gpurun_out/r2_host_phases_cfg2_v3.txt 2>&1; cat gpurun_out/r2_host_phases_cfg2_v3.txt
MSG_HOST_PHASES=1 timeout 300 python tools/prof_replay.py cfg4 2 > gpurun_out/r2_host_phases_cfg4_v3.txt 2>&1; cat gpurun_out/r2_host_phases_cfg4_v3.txt
timeout 300 python tools/prof_replay.py cfg1 3 2>&1 | tail -1; timeout 300 python tools/prof_replay.py cfg3 3 2>&1 | tail -1
timeout 600 python tools/prof_replay.py frag 2 2>&1 | tail -1
