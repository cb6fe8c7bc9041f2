# one representative K2 fw_phase3<float> launch (time-median of road1m_k256's K2: launch 465 of 501)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fw_phase3 -s 465 -c 1 -o gpurun_out/s5c_fw_phase3_f32 python bench.py --config road1m_k256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5c_ncu_p3.log 2>&1
