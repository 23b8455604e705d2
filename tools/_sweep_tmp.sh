set -u
for w in config2 config1; do for st in 1 0; do
echo "== $w static=$st"
LSDF_TUNE_STATIC=$st python tools/cycle_parts.py --flush --n 600 --workload $w | grep -v "^{" | grep "cycle graph mean"
done; done
