set -x
nvidia-smi --query-gpu=name,clocks.sm,memory.total --format=csv
free -g; nproc; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_execute.py -x -q -m gpu 2>&1 | tail -5
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_ref_cfg4.json 2> gpurun_out/r2_ref_cfg4.err
timeout 1500 python bench.py > gpurun_out/r2_bench_cfg4.json 2> gpurun_out/r2_bench_cfg4.err
timeout 900 python bench.py --config frag --steps 3 --warmup 1 --skip-cfg2 --skip-e2e --cpu-budget-s 30 > gpurun_out/r2_bench_frag.json 2> gpurun_out/r2_bench_frag.err
tail -3 gpurun_out/*.err
