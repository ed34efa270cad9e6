set -u
O=gpurun_out/s3t
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 600 python tools/ms_devtime.py cfg1 cfg3 cfg2 cfg4 frag --reps 4 > $O/planonly_devtime.jsonl 2>&1
cat $O/planonly_devtime.jsonl
