# K2 tile packing: GPU suite, full-size parity (cfg2, cfg3), bench lines
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3e_pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/s3e_pytest_gpu.log
PSP_FW_PROFILE=1 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/s3e_cfg2.json 2> gpurun_out/s3e_cfg2.err
PSP_FW_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 > gpurun_out/s3e_cfg3.json 2> gpurun_out/s3e_cfg3.err
PSP_LARGE_CONFIGS=delaunay262k_k256,delaunay1m_k1024 timeout 2000 python -m pytest tests/test_large_configs.py -m gpu -q -s > gpurun_out/s3e_large.log 2>&1; echo exit=$? >> gpurun_out/s3e_large.log
