# cfg4 spill A/B on one B200: component tables dropped + recomputed (default) vs parked on the host
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "spill or k2_order" > gpurun_out/s4a_pytest.log 2>&1; echo pytest_exit=$? >> gpurun_out/s4a_pytest.log
PSP_FW_PROFILE=1 timeout 900 python bench.py --config road4m_k512 --no-cpu-baseline > gpurun_out/s4a_cfg4_recompute.json 2> gpurun_out/s4a_cfg4_recompute.err
PSP_K2_SPILL=host PSP_FW_PROFILE=1 timeout 900 python bench.py --config road4m_k512 --no-cpu-baseline --steps 5 > gpurun_out/s4a_cfg4_host.json 2> gpurun_out/s4a_cfg4_host.err
free -g >> gpurun_out/s4a_cfg4_host.err; nproc >> gpurun_out/s4a_cfg4_host.err
