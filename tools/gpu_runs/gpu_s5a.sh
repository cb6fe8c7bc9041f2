# Component-phase wall-clock breakdown at cfg2 (3 bench runs), host alloc latency probe
mkdir -p gpurun_out
nvcc -O2 -o /tmp/alloc_probe tools/alloc_probe.cu && timeout 120 /tmp/alloc_probe > gpurun_out/s5a_alloc.txt 2>&1
for i in 1 2 3; do
  PSP_FW_PROFILE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5a_bench$i.json 2> gpurun_out/s5a_bench$i.err
done
