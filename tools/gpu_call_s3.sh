set -u
O=gpurun_out/s3r
mkdir -p $O
timeout 300 python tools/cw_phase_replay.py frag > $O/cw.txt 2>&1
head -11 $O/cw.txt
timeout 600 python -m pytest tests/test_gpu_facade.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "reorder or class_table or general_kernels or fragmented" > $O/focus.log 2>&1; tail -1 $O/focus.log
