# balanced query items + K2 timing window: GPU suite, bench lines, allocation latency probe
./tools/alloc_probe > gpurun_out/s3d_alloc.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3d_pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/s3d_pytest_gpu.log
for i in 1 2; do
PSP_FW_PROFILE=1 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/s3d_cfg2_$i.json 2> gpurun_out/s3d_cfg2_$i.err
done
PSP_FW_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 > gpurun_out/s3d_cfg3.json 2> gpurun_out/s3d_cfg3.err
./tools/alloc_probe > gpurun_out/s3d_alloc2.txt 2>&1
