timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r2_pytest_gpu14.txt 2>&1; tail -3 gpurun_out/r2_pytest_gpu14.txt
timeout 300 python tools/mc_cta_replay.py cfg2 | tail -2
timeout 300 python tools/mc_warp_replay.py cfg2
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 2 --skip-e2e --skip-execute --skip-large --skip-frag --no-migrate > gpurun_out/r2_bench_cfg2_po14.jsonl 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg2_po14.jsonl').read()); r=d['roofline']; print(d['ms_per_step'], r['frac'], r['avg_launch_ms'], r['device_timed'])"
