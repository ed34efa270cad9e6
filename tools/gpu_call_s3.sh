set -u
O=gpurun_out/s3l
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_facade.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "reorder or class_table or list_ops or general_kernels or fragmented" > $O/focus.log 2>&1; tail -2 $O/focus.log
timeout 300 python tools/cw_phase_replay.py frag > $O/cw.txt 2>&1
timeout 600 python tools/ms_devtime.py frag --reps 3 > $O/walls.txt 2>&1
cat $O/cw.txt $O/walls.txt
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
