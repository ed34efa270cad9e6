set -u
O=gpurun_out/s3u
mkdir -p $O
timeout 120 tools/bin/rp > $O/rp.txt 2>&1; cat $O/rp.txt
timeout 600 python -m pytest tests/test_gpu_facade.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "reorder or class_table or general_kernels or fragmented" > $O/focus.log 2>&1; tail -1 $O/focus.log
timeout 300 python tools/cw_phase_replay.py frag > $O/cw.txt 2>&1; cat $O/cw.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 600 python tools/ms_devtime.py frag cfg2 --reps 3 > $O/walls.txt 2>&1; cat $O/walls.txt
