timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2_pytest_gpu16.txt 2>&1; tail -3 gpurun_out/r2_pytest_gpu16.txt; grep -E "^FAILED" gpurun_out/r2_pytest_gpu16.txt | head
timeout 300 python tools/predict_latency.py
timeout 300 python tools/ingest_bench.py 2>&1 | tail -8
