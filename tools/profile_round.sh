#!/bin/bash
# Round-end evidence set, run on the GPU box under gpurun:
#   gpurun --timeout 3000 -- 'bash tools/profile_round.sh'
# GPU tests + smoke, launch lists (plan-only and migrating cfg2 replays),
# ncu --set full captures of the multisplit at cfg2 and cfg4, the default
# bench line and the reference arm.  Outputs land in gpurun_out/.
set -u
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
tail -1 $O/smoke.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2_planonly.csv \
    python tools/prof_replay.py cfg2 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2_migrate.csv \
    python tools/prof_replay.py cfg2 1 --migrate > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -f -k regex:k_ms_coop -s 40 -c 1 -o $O/ncu_coop_cfg2 \
    python tools/prof_replay.py cfg2 1 > /dev/null 2>&1
ncu --set full --clock-control none -f -k regex:k_ms_coop -s 100 -c 1 -o $O/ncu_coop_cfg4 \
    python tools/prof_replay.py cfg4 1 > /dev/null 2>&1
timeout 300 python tools/um_time.py > $O/um_time.txt 2>&1; tail -1 $O/um_time.txt
timeout 300 python tools/ms_probe.py cfg2 3 > $O/ms_probe.txt 2>&1; timeout 300 python tools/ms_probe.py cfg4 2 >> $O/ms_probe.txt 2>&1
tail -2 $O/ms_probe.txt
timeout 1200 python bench.py > $O/bench.jsonl 2> $O/bench.err; tail -c 400 $O/bench.jsonl
timeout 900 python bench.py --impl reference > $O/bench_ref.jsonl 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.jsonl
