set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2_pytest_gpu4.txt 2>&1; tail -8 gpurun_out/r2_pytest_gpu4.txt
timeout 300 python tools/mc_cta_replay.py cfg2 > gpurun_out/r2_mc_cta_cfg2_v2.txt 2>&1; tail -4 gpurun_out/r2_mc_cta_cfg2_v2.txt
timeout 600 python tools/prof_replay.py frag 2 > gpurun_out/r2_frag_replay_v2.txt 2>&1; cat gpurun_out/r2_frag_replay_v2.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_frag_v2.csv python tools/prof_replay.py frag 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_launches_frag_v2.csv > gpurun_out/r2_launches_frag_v2_summary.txt 2>&1; cat gpurun_out/r2_launches_frag_v2_summary.txt
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 2 --skip-e2e --skip-execute --skip-large --no-migrate > gpurun_out/r2_bench_cfg2_planonly.json 2>gpurun_out/r2_bench_cfg2_planonly.err; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg2_planonly.json').read()); print(d['ms_per_step'], json.dumps(d['roofline']))"
