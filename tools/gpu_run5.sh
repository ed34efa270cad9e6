set -x
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider "tests/test_gpu_facade.py::test_large_reorder_matches_closed_form" "tests/test_gpu_parity.py::test_general_kernels_match_reference[llm_2.0]" "tests/test_gpu_parity.py::test_gpu_matches_reference[frag_s-ideal]" > gpurun_out/r2_sanitize5.txt 2>&1; echo "sanitize rc=$?"; grep -E "Invalid|ERROR SUMMARY|passed|failed" gpurun_out/r2_sanitize5.txt | head -20
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2_pytest_gpu5.txt 2>&1; tail -12 gpurun_out/r2_pytest_gpu5.txt
timeout 300 python tools/mc_cta_replay.py cfg2 > gpurun_out/r2_mc_cta_cfg2_v3.txt 2>&1; tail -3 gpurun_out/r2_mc_cta_cfg2_v3.txt
timeout 600 python tools/prof_replay.py frag 2 > gpurun_out/r2_frag_replay_v3.txt 2>&1; cat gpurun_out/r2_frag_replay_v3.txt
