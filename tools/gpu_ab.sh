timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
for p in default 8x8; do PSP_QUERY_PRODUCT=$p timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err; done
PSP_QUERY_PRODUCT=default timeout 400 python bench.py --no-cpu-baseline --config delaunay1m_k1024 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
