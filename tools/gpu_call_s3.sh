set -u
O=gpurun_out/s3s
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python tools/ms_devtime.py cfg1 cfg3 cfg2 cfg4 frag --reps 4 > $O/planonly_devtime.jsonl 2>&1
cat $O/planonly_devtime.jsonl
timeout 300 python tools/cw_phase_replay.py frag > $O/cw.txt 2>&1
