set -u
O=gpurun_out/s3i
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_facade.py -q -x -p no:cacheprovider > $O/facade.log 2>&1; tail -2 $O/facade.log
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python tools/cw_phase_replay.py frag > $O/cw.txt 2>&1
timeout 600 python tools/ms_devtime.py cfg1 cfg3 cfg2 cfg4 frag --reps 3 > $O/walls.txt 2>&1
for c in cfg2 cfg4; do timeout 300 python tools/mc_phase_replay.py $c; done > $O/mc.txt 2>&1
cat $O/cw.txt $O/walls.txt $O/mc.txt
