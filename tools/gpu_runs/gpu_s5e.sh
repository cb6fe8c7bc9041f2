# small-buffer cache (budgets count cached bytes, no flush): full GPU suite, smoke, cfg2 bench x2 (component laps), cfg4 bench (memory-tight path)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5e_pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/s5e_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5e_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/s5e_smoke.log
for i in 1 2; do
  PSP_FW_PROFILE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s5e_bench$i.json 2> gpurun_out/s5e_bench$i.err
done
PSP_FW_PROFILE=1 timeout 1200 python bench.py --config road4m_k512 --no-cpu-baseline > gpurun_out/s5e_cfg4.json 2> gpurun_out/s5e_cfg4.err
