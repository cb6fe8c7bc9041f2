# cfg4 (road 2048^2, f32) bench + full-size parity
grep MemAvailable /proc/meminfo > gpurun_out/meminfo.txt; nvidia-smi --query-gpu=memory.total --format=csv >> gpurun_out/meminfo.txt
PSP_FW_PROFILE=1 timeout 1200 python bench.py --no-cpu-baseline --config road4m_k512 > gpurun_out/bench_road.json 2> gpurun_out/bench_road.err
PSP_LARGE_CONFIGS=road4m_k512 timeout 1500 python -m pytest tests/test_large_configs.py -m gpu -q -s > gpurun_out/large.log 2>&1
