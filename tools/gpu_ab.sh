# A/B driver for gpurun: GPU tests, then bench variants (JSON in gpurun_out/)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
