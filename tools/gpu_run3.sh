set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_msim_plugin.py tests/test_gpu_abi_errors.py -q -m gpu -p no:cacheprovider -x > gpurun_out/r2_pytest_plugin.txt 2>&1; tail -5 gpurun_out/r2_pytest_plugin.txt
timeout 300 python tools/mc_cta_replay.py cfg2 > gpurun_out/r2_mc_cta_cfg2.txt 2>&1; cat gpurun_out/r2_mc_cta_cfg2.txt
timeout 300 python tools/host_profile.py > gpurun_out/r2_host_profile_cfg2.txt 2>&1; cat gpurun_out/r2_host_profile_cfg2.txt
timeout 300 python tools/py_profile.py > gpurun_out/r2_py_profile_cfg2.txt 2>&1; head -40 gpurun_out/r2_py_profile_cfg2.txt
timeout 300 python tools/predict_latency.py > gpurun_out/r2_predict_latency.txt 2>&1; cat gpurun_out/r2_predict_latency.txt
