timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r2_pytest_gpu20.txt 2>&1; tail -3 gpurun_out/r2_pytest_gpu20.txt; grep -E "^FAILED|^E " gpurun_out/r2_pytest_gpu20.txt | head
for c in cfg2 cfg4; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_v20.csv python tools/prof_replay.py $c 1 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_${c}_v20.csv | head -8; done
timeout 300 python tools/prof_replay.py cfg2 3 | tail -1; timeout 300 python tools/prof_replay.py cfg4 2 | tail -1
