set -u
O=gpurun_out/s3m
mkdir -p $O
for lib in tools/bin/libmsched_prev.so paper_2512_24637_b200/libmsched_b200.so; do echo "== $lib"; MSG_LIB=$lib timeout 600 python tools/ms_devtime.py frag cfg2 cfg3 --reps 3; done > $O/walls.txt 2>&1
cat $O/walls.txt
timeout 600 python -m pytest tests/test_gpu_facade.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/focus.log 2>&1; tail -2 $O/focus.log
