for v in 1 2; do python tools/cycle_parts.py --flush --n 400 --workload config2 | grep -v "^{" | grep "^fk\|cycle graph mean"; done
python -m pytest tests/test_gpu_parity.py -q -k "fk or full_pipeline" 2>&1 | tail -1
