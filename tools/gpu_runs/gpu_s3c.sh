# K1 nested-dissection order + batched sparse walk: GPU suite, then bench lines
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3c_pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/s3c_pytest_gpu.log
PSP_FW_PROFILE=1 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/s3c_cfg2.json 2> gpurun_out/s3c_cfg2.err
PSP_FW_PROFILE=1 PSP_K1_ORDER=natural timeout 400 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/s3c_cfg2_nat.json 2> gpurun_out/s3c_cfg2_nat.err
PSP_FW_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 > gpurun_out/s3c_cfg3.json 2> gpurun_out/s3c_cfg3.err
PSP_FW_PROFILE=1 timeout 1200 python bench.py --no-cpu-baseline --config road4m_k512 > gpurun_out/s3c_cfg4.json 2> gpurun_out/s3c_cfg4.err
