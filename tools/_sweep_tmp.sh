set -u
for w in config2 config1; do for ff in 1 0; do
echo "== $w fused=$ff"
LSDF_TUNE_FUSEFIN=$ff python tools/cycle_parts.py --flush --n 400 --workload $w | grep -v "^{" | grep "cycle graph mean\|p99"
done; done
