"""Copy the evidence produced by tools/refresh_profiles.sh (gpurun_out/prof/)
into profiles/<round>/ and regenerate the ncu summary text.

    python tools/collect_profiles.py [--round r01]
"""
import argparse
import json
import shutil
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent


def write_counters(src, out_path, rnd):
    """Per-launch DRAM traffic and warp instructions of the query kernel (read by bench.py's rooflines)."""
    import csv

    traffic = {}
    for w in ("config4", "config2"):
        out = subprocess.run(["ncu", "-i", str(src / f"shells_{w}.ncu-rep"), "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout.splitlines()
        rows = list(csv.reader(out))
        h, u, v = rows[0], rows[1], rows[2]
        d = dict(zip(h, zip(u, v)))

        def val(k):
            unit, x = d[k]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return float(x.replace(",", "")) * scale

        traffic[w] = int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
        traffic[f"{w}_warp_inst"] = int(val("smsp__inst_executed.sum"))
    traffic["_units"] = ("bytes per launch of query_shells_kernel: dram__bytes_read.sum + dram__bytes_write.sum from "
                         f"one ncu --set full capture (profiles/{rnd}/ncu_summary.txt); <w>_warp_inst: "
                         "smsp__inst_executed.sum of the same launch")
    Path(out_path).write_text(json.dumps(traffic))
    return traffic


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--counters-only", metavar="OUT", help="write the query counters JSON to OUT and stop")
    args = ap.parse_args()
    src = REPO / "gpurun_out" / "prof"
    if args.counters_only:
        print(write_counters(src, args.counters_only, args.round))
        return
    dst = REPO / "profiles" / args.round
    dst.mkdir(parents=True, exist_ok=True)
    for a, b in (("bench.json", "bench_config4_N1.json"), ("bench_config2.json", "bench_config2_N1.json"),
                 ("bench_reference.json", "bench_reference_port.json")):
        line = (src / a).read_text().strip().splitlines()[-1]
        json.loads(line)
        (dst / b).write_text(line + "\n")
    for f in ("launches_config4.csv", "launches_config2.csv", "launches_bench.csv"):
        shutil.copy(src / f, dst / f)
    for a, b in (("config5_dynamic.json", "config5_dynamic.json"), ("vmajor_config2.json", "vmajor_config2.json"),
                 ("vmajor_config5.json", "vmajor_config5.json"), ("config3_precompute.json", "config3_precompute.json"),
                 ("scan_stats.txt", "scan_stats.txt")):
        if (src / a).exists() and (src / a).stat().st_size > 0:
            shutil.copy(src / a, dst / b)
    traffic = write_counters(src, REPO / "profiles" / "query_traffic.json", args.round)
    py = sys.executable
    lines = [f"# ncu summaries, round {args.round[1:]} (tools/refresh_profiles.sh; B200, --clock-control none)", "",
             "## launch lists (cold, serialised; the first 4 query launches of each process are the checker's "
             "warm-up with an empty cloud; the bench list includes the 256 MiB L2-flush fills)"]
    for f in ("launches_bench", "launches_config4", "launches_config2"):
        r = subprocess.run([py, str(REPO / "tools" / "ncu_launches.py"), str(src / f"{f}.csv")],
                           capture_output=True, text=True).stdout.splitlines()
        lines += [f"### {f}.csv"] + r[1:9]
    for w in ("config4", "config2"):
        lines += ["", f"## query_shells_kernel, {w} (ncu --set full, the first real query launch)"]
        r = subprocess.run([py, str(REPO / "tools" / "ncu_summary.py"), str(src / f"shells_{w}.ncu-rep")],
                           capture_output=True, text=True).stdout.splitlines()
        lines += r[1:]
        lines += ["", "### hottest source lines"]
        r = subprocess.run([py, str(REPO / "tools" / "ncu_lines.py"), str(src / f"shells_{w}.ncu-rep"), "25"],
                           capture_output=True, text=True).stdout.splitlines()
        lines += r
    (dst / "ncu_summary.txt").write_text("\n".join(lines) + "\n")
    print("collected into", dst, traffic)


if __name__ == "__main__":
    main()
