# round 2: A/B driver warm-up during the host partition (bench x3 each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do
for w in 0 1; do
if [ $w = 1 ]; then export PSP_WARM_DRIVER=1; else unset PSP_WARM_DRIVER; fi
timeout 1200 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2bc_$i$w.json 2> gpurun_out/r2bc_$i$w.err
python -c "import json;d=json.load(open('gpurun_out/r2bc_$i$w.json'));p=d['preprocessing'];print('warm=$w', p['preprocessing_s'], p['partition_s'], p['component_apsp_s'], p['boundary_minus_k2_device_s'], p['driver_alloc'])"
done
done
