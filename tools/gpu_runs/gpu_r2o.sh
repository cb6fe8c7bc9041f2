# round 2: small-batch kernels at cfg3: launch lists (1K, grouped and cta) + ncu of query_cta
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for kn in grouped cta; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2o_list_$kn.csv python tools/profile_query.py --config delaunay1m_k1024 --batch 1000 --batches 4 --kernel $kn > gpurun_out/r2o_$kn.log 2>&1; echo $kn rc=$?
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:query_cta --launch-skip 2 --launch-count 1 -o gpurun_out/r2o_cta_1k python tools/profile_query.py --config delaunay1m_k1024 --batch 1000 --batches 4 --kernel cta > gpurun_out/r2o_ncu.log 2>&1; echo ncu rc=$?
python tools/profile_query.py --config delaunay1m_k1024 --batch 1000 --batches 6 --kernel cta
python tools/profile_query.py --config delaunay1m_k1024 --batch 1000 --batches 6 --kernel grouped
