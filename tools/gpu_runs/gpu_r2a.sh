set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
free -g; nproc
python -m pytest tests/test_gpu_parity.py -k "tile_packed" -x -q 2>&1 | tail -5
timeout 900 ./oracle/_ref/shim/gpu_acceptance > gpurun_out/acc1.log 2>&1; echo acc_rc=$?
tail -12 gpurun_out/acc1.log
timeout 1200 python -m pytest tests/test_large_configs.py -x -q -s 2>&1 | tail -8
