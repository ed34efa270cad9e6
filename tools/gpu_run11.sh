timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_facade.py "tests/test_gpu_parity.py::test_general_kernels_match_reference" "tests/test_gpu_parity.py::test_fragmented_migration_uses_the_gather_kernel" -k "not cfg4" > gpurun_out/r2_pytest_gpu11.txt 2>&1; tail -3 gpurun_out/r2_pytest_gpu11.txt; grep -E "^FAILED|^E " gpurun_out/r2_pytest_gpu11.txt | head
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "frag" > gpurun_out/r2_pytest_gpu11b.txt 2>&1; tail -3 gpurun_out/r2_pytest_gpu11b.txt
timeout 600 python tools/prof_replay.py frag 2 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_frag_v5.csv python tools/prof_replay.py frag 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_launches_frag_v5.csv | head -8
