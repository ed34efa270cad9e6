timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r2_pytest_gpu18.txt 2>&1; tail -3 gpurun_out/r2_pytest_gpu18.txt; grep -E "^FAILED|^E " gpurun_out/r2_pytest_gpu18.txt | head
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --skip-e2e --skip-execute --skip-large --skip-frag --skip-cfg2 --no-migrate > gpurun_out/r2_bench_cfg4_po.jsonl 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg4_po.jsonl').read()); r=d['roofline']; print(d['ms_per_step'], r['frac'], r['avg_launch_ms'], r['device_timed'])"
timeout 600 python tools/ms_bench.py 2>&1 | tail -6
