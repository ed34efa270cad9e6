O=gpurun_out/p9; mkdir -p $O
timeout 300 python tools/predict_latency.py > $O/predict_latency.txt 2>&1; cat $O/predict_latency.txt
timeout 1200 python -m pytest tests/test_gpu_facade.py tests/test_gpu_predictor_edges.py tests/test_gpu_acceptance.py -x -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -4 $O/gpu_tests.log
