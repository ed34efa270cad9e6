set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2_pytest_gpu.txt 2>&1; tail -15 gpurun_out/r2_pytest_gpu.txt
timeout 600 python bench.py --config cfg2 --steps 3 --warmup 1 --skip-e2e --skip-plan-only --skip-large > gpurun_out/r2_bench_cfg2_exec.json 2> gpurun_out/r2_bench_cfg2_exec.err
timeout 600 python tools/prof_replay.py frag 2 > gpurun_out/r2_frag_replay.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_frag.csv python tools/prof_replay.py frag 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_launches_frag.csv > gpurun_out/r2_launches_frag_summary.txt 2>&1
cat gpurun_out/r2_frag_replay.txt gpurun_out/r2_launches_frag_summary.txt
