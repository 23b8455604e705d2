for i in 1 2; do
for v in 0 1; do
LSDF_TUNE_LDS=$v python bench.py --steps 30 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); r=d['roofline']; print('LDS=$v', round(r['kernel_ms']*1000,1), 'us', int(r['warp_inst_per_launch']), round(r['frac'],3), 'value', round(d['value']/1e6,1), 'c2 p50/p99', round(d['realtime']['device_p50_us'],2), round(d['realtime']['device_p99_us'],2))"
done; done
