#!/bin/bash
# compute-sanitizer passes over the CUDA path (run on the GPU box under gpurun):
#   gpurun --timeout 2400 -- 'bash tools/sanitize.sh'
# memcheck on golden replays (fast paths and, via MSG_FALLBACK, the general
# kernels) and a full cfg2 replay; racecheck and synccheck on the facade's
# reorder tests (the cooperative multisplit, the fused window kernel);
# initcheck on golden replays.
set -u
O=gpurun_out/sanitize.txt
: > $O
run() {
  echo "### $*" >> $O
  timeout 1200 "$@" > /tmp/san.log 2>&1
  grep -E "passed|failed|rep 0|SUMMARY" /tmp/san.log | tail -3 >> $O
}
CS="compute-sanitizer --print-limit 20"
run $CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_facade.py -x -q \
    -k "stream_2.0 or frag or opt_3 or llm_1.5 or struct or madvise or reorder or evict or plan_migration"
MSG_FALLBACK=windows,onesweep,demand run $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -x -q \
    -k "cfg3_2.0 or frag"
run $CS --tool memcheck python tools/prof_replay.py cfg2 1
run $CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_execute.py -x -q \
    -k "(moves_the_right_bytes and (stream_3.0 or llm_2.0 or frag)) or executed or execute_needs"
run $CS --tool memcheck python -m pytest tests/test_gpu_abi_errors.py tests/test_gpu_tracebin.py -x -q
run $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -x -q -k "moves_the_right_bytes and (stream_3.0 or frag)"
run $CS --tool initcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_facade.py -x -q \
    -k "(test_gpu_matches and (stream_2.0 or llm_1.5 or edge_tiny or frag)) or madvise or plan_migration or (moves_the_right_bytes and stream_3.0)"
run $CS --tool racecheck python -m pytest tests/test_gpu_facade.py -x -q -k "multi_window or large_reorder or randomized"
run $CS --tool synccheck python -m pytest tests/test_gpu_facade.py -x -q -k "multi_window or large_reorder"
# the async switch path (k_switch_coop: plan, multisplit and apply as phases of one cooperative launch)
run $CS --tool racecheck python -m pytest tests/test_gpu_engine.py -x -q -k "async"
run $CS --tool synccheck python -m pytest tests/test_gpu_engine.py -x -q -k "async"
run $CS --tool initcheck python -m pytest tests/test_gpu_engine.py -x -q -k "async"
run $CS --tool memcheck python -m pytest tests/test_gpu_engine.py tests/test_gpu_msim_plugin.py -x -q
# late round 2: the queued per-entry chunks of the multisplit, the grouped class-table keys, the radix-sorted
# window runs (general kernels forced by MSG_FALLBACK on the fragmented goldens)
run $CS --tool racecheck python -m pytest tests/test_gpu_facade.py -x -q -k "class_table_groups or multi_window"
MSG_FALLBACK=windows,demand run $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -x -q -k "general_kernels and frag"
MSG_FALLBACK=windows,demand run $CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_facade.py -x -q -k "frag or class_table_groups or large_reorder"
run $CS --tool synccheck python -m pytest tests/test_gpu_facade.py -x -q -k "class_table_groups"
cat $O
