set -u
O=gpurun_out/s3f
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
for c in cfg1 cfg3 cfg2 cfg4 frag; do echo "== $c"; MSG_LIB=tools/bin/libmsched_old.so timeout 300 python tools/ms_devtime.py $c --reps 4; timeout 300 python tools/ms_devtime.py $c --reps 4; done > $O/walls.txt 2>&1
for c in cfg1 cfg2; do echo "== $c"; timeout 300 python tools/host_profile.py $c; done > $O/hostprof.txt 2>&1
MSG_HOST_PHASES=1 timeout 300 python tools/prof_replay.py cfg2 3 > $O/host_phases_cfg2.txt 2>&1
cat $O/walls.txt $O/hostprof.txt $O/host_phases_cfg2.txt
