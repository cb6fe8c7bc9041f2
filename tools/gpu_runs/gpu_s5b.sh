# f32 tolerance path evidence at a size ncu can replay: road1m_k256 bench line, then one
# fw_phase3 launch inside K2 and one query_grouped launch under ncu --set full
mkdir -p gpurun_out
PSP_FW_PROFILE=1 timeout 900 python bench.py --config road1m_k256 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s5b_road1m.json 2> gpurun_out/s5b_road1m.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/s5b_road1m_launches.csv python bench.py --config road1m_k256 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s5b_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fw_phase3 -s 200 -c 1 -o gpurun_out/s5b_fw_phase3_f32 python bench.py --config road1m_k256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5b_ncu_p3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_grouped -s 2 -c 1 -o gpurun_out/s5b_query_grouped_f32 python bench.py --config road1m_k256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5b_ncu_qg.log 2>&1
