#!/bin/bash
# Round-2 evidence set, run on the GPU box under gpurun:
#   gpurun --timeout 5400 -- 'bash tools/profile_round2.sh'
# GPU tests + smoke, the default bench line (config 4) and the reference arm,
# launch lists (cfg4 / cfg2 / fragmented), ncu --set full captures of every
# planner kernel at config 4 and of the multisplit at config 2, the host
# phase clock.  Outputs land in gpurun_out/r02/.
set -u
O=gpurun_out/r02
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
tail -1 $O/smoke.log
timeout 900 python bench.py --impl reference > $O/bench_ref.jsonl 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.jsonl
timeout 2400 python bench.py > $O/bench.jsonl 2> $O/bench.err; tail -c 400 $O/bench.jsonl
for cfg in cfg4 cfg2 frag; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${cfg}_planonly.csv \
      python tools/prof_replay.py $cfg 1 > /dev/null 2>&1
  python tools/launch_summary.py $O/launches_${cfg}_planonly.csv > $O/launches_${cfg}_planonly_summary.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2_migrate.csv \
    python tools/prof_replay.py cfg2 1 --migrate > /dev/null 2>&1
python tools/launch_summary.py $O/launches_cfg2_migrate.csv > $O/launches_cfg2_migrate_summary.txt
for k in k_windows_fused k_switch_coop k_ranges_from_iv; do
  timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:$k -s 30 -c 1 -o $O/ncu_${k}_cfg4 \
      python tools/prof_replay.py cfg4 1 > /dev/null 2>&1
done
# the standalone multisplit launches of the migrating (headline) replay; several consecutive ones
timeout 1800 ncu --set full --import-source on --clock-control none -f -k regex:k_ms_coop -s 30 -c 4 -o $O/ncu_k_ms_coop_cfg4 \
    python tools/prof_replay.py cfg4 1 --migrate > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:k_ms_coop -s 40 -c 1 -o $O/ncu_k_ms_coop_cfg2 \
    python tools/prof_replay.py cfg2 1 --migrate > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:k_switch_coop -s 40 -c 1 -o $O/ncu_k_switch_coop_cfg2 \
    python tools/prof_replay.py cfg2 1 > /dev/null 2>&1
for k in k_window_combine_wide k_window_runs k_switch_coop; do
  timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:$k -s 200 -c 1 -o $O/ncu_${k}_frag \
      python tools/prof_replay.py frag 1 > /dev/null 2>&1
done
# device phase stamps (the phase-timing build, tools/bin/libmsched_mcts.so: `make phase-ts` before the call)
for c in cfg2 cfg4 cfg1; do timeout 300 python tools/sw_phase_replay.py $c; done > $O/switch_kernel_phases.txt 2>&1
for c in cfg2 cfg4 cfg1; do timeout 300 python tools/fw_phase_replay.py $c; done > $O/window_kernel_phases.txt 2>&1
for c in cfg1 cfg3 cfg2 cfg4; do echo "== $c"; timeout 300 python tools/prof_replay.py $c 4; done > $O/planonly_all.txt 2>&1
timeout 600 python tools/ms_devtime.py cfg1 cfg3 cfg2 cfg4 frag --reps 4 > $O/planonly_devtime.jsonl 2>&1
timeout 300 python tools/cw_phase_replay.py frag > $O/frag_window_phases.txt 2>&1
for c in cfg2 cfg4; do timeout 300 python tools/mc_cta_replay.py $c | tail -3; done > $O/multisplit_cta_phases.txt 2>&1
MSG_HOST_PHASES=1 timeout 300 python tools/prof_replay.py cfg2 3 > $O/host_phases_cfg2.txt 2>&1
MSG_HOST_PHASES=1 timeout 300 python tools/prof_replay.py cfg4 2 > $O/host_phases_cfg4.txt 2>&1
timeout 300 python tools/predict_latency.py > $O/predict_latency.txt 2>&1
ls -la $O
