# 1-GPU result collection for DESIGN/README (JSON lines into gpurun_out/)
timeout 900 python bench.py > gpurun_out/c1_cfg2.json 2> gpurun_out/c1_cfg2.err
PSP_FW_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 > gpurun_out/c1_cfg3.json 2> gpurun_out/c1_cfg3.err
PSP_FW_PROFILE=1 timeout 1200 python bench.py --no-cpu-baseline --config road4m_k512 > gpurun_out/c1_cfg4.json 2> gpurun_out/c1_cfg4.err
timeout 1200 python tools/query_sweep.py > gpurun_out/c1_sweep.jsonl 2> gpurun_out/c1_sweep.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/c1_ref.json 2> gpurun_out/c1_ref.err
