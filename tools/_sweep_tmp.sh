set -u
for v in "1 1" "0 0" "1 0" "0 1" "1 1"; do set -- $v
echo "== fkreset=$1 occclear=$2"
LSDF_TUNE_FKRESET=$1 LSDF_TUNE_OCCCLEAR=$2 python tools/cycle_parts.py --flush --n 600 --workload config2 | grep -v "^{" | grep "cycle graph mean"
done
