# One GPU call that regenerates the round's evidence under gpurun_out/prof/.
#   gpurun -- 'bash tools/refresh_profiles.sh'      then   python tools/collect_profiles.py --round r02
set -u
O=gpurun_out/prof
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 300 $O/bench_reference.json
# launch list of the bench command (cold, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-counters > $O/ncu_bench.log 2>&1
# one full capture per workload of the scan (the bench's probe cycle) and of the whole config-2 cycle
for w in config4 config2; do
  ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:query_shells -f \
      -o $O/shells_$w python bench.py --probe-counters --workload $w > $O/ncu_full_$w.log 2>&1
done
ncu --set full --import-source on --clock-control none --profile-from-start off -f -o $O/cycle_config2 \
    python bench.py --probe-counters --workload config2 > $O/ncu_cycle_config2.log 2>&1
python tools/scan_stats.py build > /dev/null 2>&1 && python tools/scan_stats.py config2 config4 > $O/scan_stats.txt 2>&1
python tools/scan_timing.py build > /dev/null 2>&1 && python tools/scan_timing.py config2 config1 > $O/scan_timing.txt 2>&1
python tools/cycle_parts.py --workload config2 --flush > $O/cycle_parts_config2.txt 2>&1
python tools/e2e_breakdown.py > $O/e2e_breakdown_config2.txt 2>&1
python tools/bench_vmajor.py --workload config2 > $O/vmajor_config2.json 2> $O/vmajor.err
python tools/bench_vmajor.py --workload config5 > $O/vmajor_config5.json 2>> $O/vmajor.err
python tools/bench_precompute.py --train --placement > $O/config3_precompute.json 2> $O/config3_precompute.err
# neural placement at config-3 scale: the fused MLP + sampler kernel vs the two-kernel path
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active \
    -k regex:"mlp_place_tc|place_windows|fill_masked|layer1_pack|mlp_tc_kernel" --clock-control none --csv \
    --log-file $O/placement_launches.csv python tools/bench_precompute.py --placement > $O/ncu_placement.log 2>&1
python tools/reference_tests.py run > $O/reference_tests.log 2>&1; cp gpurun_out/reference_tests.txt $O/ 2>/dev/null
echo done
