"""Key counters of one ncu --set full report (first profiled kernel)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    for v in r[2:]:
        d = dict(zip(h, v))
        print(f" [{d.get('Kernel Name', '?')[:70]}]")
        for k in KEYS:
            if k in d:
                print(f"  {k:62s} {d[k]}")
        stalls = {k: float(d[k].replace(",", "")) for k in h
                  if "issue_stalled" in k and k.endswith("per_issue_active.ratio") and d.get(k)}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        print("  stalls/issue: " + ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={x:.2f}" for k, x in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        main(p)
