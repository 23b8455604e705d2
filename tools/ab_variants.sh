# A/B on one box: each argument is `base`, a library variant built with
# tools/build_variant.py into paper_2309_12543_b200/_lib/ (`var_b.so`), or an
# environment assignment for the base library (`LSDF_TUNE_PAIR=0`).
#   bash tools/ab_variants.sh base var_b.so LSDF_TUNE_PAIR=0
for i in 1 2; do
for v in "$@"; do
(
case "$v" in
  base) ;;
  *=*) export "$v" ;;
  *) export LINKSDF_B200_LIB=paper_2309_12543_b200/_lib/$v ;;
esac
python bench.py --steps 30 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; print('$v', round(r['kernel_ms']*1000,1), 'us', int(r['warp_inst_per_launch']), round(r['frac'],3), 'value', round(d['value']/1e6,1), 'c2 p50/p99', round(d['realtime']['device_p50_us'],2), round(d['realtime']['device_p99_us'],2), 'e2e', round(d['e2e']['value']/1e6,1))"
)
done; done
