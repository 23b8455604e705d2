# A/B of library variants / tuning overrides with the config-4 cloud variants (crowd, empty, far corners, sparse)
# and the config-1/2 latency: bash tools/ab_clouds.sh base var_x.so   (variants as in tools/ab_variants.sh)
for v in "$@"; do
(
case "$v" in base) ;; *=*) export "$v" ;; *) export LINKSDF_B200_LIB=paper_2309_12543_b200/_lib/$v ;; esac
python bench.py --steps 30 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; cv=d['cloud_variants']
print('$v', round(r['kernel_ms']*1000,1), 'us', int(r['warp_inst_per_launch']), 'value', round(d['value']/1e6,1), {k: round(v['ms_per_step']*1000,1) for k,v in cv.items()}, 'c2', round(d['realtime']['device_p50_us'],2), 'c1', round(d['config1']['device_p50_us'],2))"
)
done
