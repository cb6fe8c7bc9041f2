# round-1 final 1-GPU collection: suite, bench lines (cfg2 with CPU baseline, cfg3, cfg4), reference arm, ncu
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3g_pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/s3g_pytest_gpu.log
PSP_FW_PROFILE=1 timeout 900 python bench.py > gpurun_out/s3g_cfg2.json 2> gpurun_out/s3g_cfg2.err
PSP_FW_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 > gpurun_out/s3g_cfg3.json 2> gpurun_out/s3g_cfg3.err
PSP_FW_PROFILE=1 timeout 1200 python bench.py --no-cpu-baseline --config road4m_k512 > gpurun_out/s3g_cfg4.json 2> gpurun_out/s3g_cfg4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s3g_ref.json 2> gpurun_out/s3g_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3g_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s3g_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_grouped -s 2 -c 1 -o gpurun_out/s3g_query_grouped python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s3g_ncu_qg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fw_phase3 -s 280 -c 1 -o gpurun_out/s3g_fw_phase3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s3g_ncu_p3.log 2>&1
