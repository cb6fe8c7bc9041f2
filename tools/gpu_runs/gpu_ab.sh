# A/B driver for gpurun: GPU tests, then bench variants (JSON in gpurun_out/)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
PSP_FW_PROFILE=1 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
PSP_FW_PROFILE=1 PSP_BG_ORDER=component timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_component.json 2> gpurun_out/bench_component.err
PSP_FW_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
PSP_LARGE_CONFIGS=delaunay262k_k256,delaunay1m_k1024,road4m_k512 timeout 2500 python -m pytest tests/test_large_configs.py -m gpu -q -s > gpurun_out/large.log 2>&1
