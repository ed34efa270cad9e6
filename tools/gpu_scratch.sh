O=gpurun_out/p7; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -4 $O/gpu_tests.log
timeout 1500 python bench.py --steps 3 --warmup 3 --skip-execute --skip-frag > $O/bench.jsonl 2> $O/bench.err; python - <<'P'
import json
d=json.loads(open("gpurun_out/p7/bench.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], json.dumps(d["roofline"])[:600])
print(json.dumps(d.get("plan_only",{}))[:500])
print(json.dumps(d.get("cfg2",{}).get("roofline",{}))[:500])
P
tail -3 $O/bench.err
