timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3_pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/s3_pytest_gpu.log
PSP_FW_PROFILE=1 timeout 600 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv >> gpurun_out/s3_bench.err
