# round 2: query_cta shapes (warps x unroll x min blocks) at 1K-10K pairs on cfg3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 7 12 13 14 15 16; do
PSP_CTA_VARIANT=$v timeout 600 python tools/query_sweep.py --config delaunay1m_k1024 --sizes 1e3,3e3,1e4,3e4 --kernels cta --no-e2e > gpurun_out/r2y_v$v.jsonl 2> gpurun_out/r2y_v$v.err
python -c "
import json
print($v, [(json.loads(l)['batch_per_gpu'], round(json.loads(l)['queries_per_s']/1e6,1)) for l in open('gpurun_out/r2y_v$v.jsonl')])"
done
