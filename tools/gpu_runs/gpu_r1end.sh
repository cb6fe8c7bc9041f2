# Round-end check on one B200: full GPU suite, smoke(), default bench line, launch list of the same bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e_pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/e_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/e_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/e_smoke.log
PSP_FW_PROFILE=1 timeout 900 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/e_ref.json 2> gpurun_out/e_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/e_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e_ncu.log 2>&1
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv >> gpurun_out/e_bench.err
