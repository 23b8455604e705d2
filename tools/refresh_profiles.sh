# One GPU call that regenerates the round's evidence under gpurun_out/prof/.
#   gpurun -- 'bash tools/refresh_profiles.sh'
set -u
O=gpurun_out/prof
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
# ncu first: the query kernel's DRAM bytes and instruction count feed the bench line's rooflines
for w in config4 config2; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv \
      python tools/profile_step.py --workload $w --device-only --steps 8 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:query_shells -s 5 -c 1 -f -o $O/shells_$w \
      python tools/profile_step.py --workload $w --device-only --steps 8 > $O/ncu_full_$w.log 2>&1
done
python tools/collect_profiles.py --counters-only profiles/query_traffic.json > $O/counters.log 2>&1
cp profiles/query_traffic.json $O/query_traffic.json
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 300 $O/bench_reference.json
python bench.py --workload config2 --no-cpu-baseline > $O/bench_config2.json 2> $O/bench_config2.err
# launch list of the bench command (cold, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
python tools/scan_stats.py config2 config4 > $O/scan_stats.txt 2>&1
echo done
# secondary workloads (configs 3 and 5, materialized mode) for DESIGN §6

python tools/bench_vmajor.py --workload config2 > $O/vmajor_config2.json 2> $O/vmajor.err
python tools/bench_vmajor.py --workload config5 > $O/vmajor_config5.json 2>> $O/vmajor.err
python tools/bench_precompute.py > $O/config3_precompute.json 2> $O/config3_precompute.err
echo done2
