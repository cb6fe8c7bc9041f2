# K2 per-k-block trace (cfg3), packed and contiguous layouts
PSP_K2_TRACE=gpurun_out/s3f_trace_pack.txt PSP_FW_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 --steps 3 > gpurun_out/s3f_pack.json 2> gpurun_out/s3f_pack.err
PSP_BG_PACK=0 PSP_K2_TRACE=gpurun_out/s3f_trace_cont.txt PSP_FW_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --config delaunay1m_k1024 --steps 3 > gpurun_out/s3f_cont.json 2> gpurun_out/s3f_cont.err
