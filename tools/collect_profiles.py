"""Copy the evidence produced by tools/refresh_profiles.sh (gpurun_out/prof/)
into profiles/<round>/ and write the ncu summary text.

    python tools/collect_profiles.py --round r02
"""
import argparse
import json
import shutil
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO / "tools"))


def _run(args):
    return subprocess.run([sys.executable, *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r02")
    args = ap.parse_args()
    src = REPO / "gpurun_out" / "prof"
    dst = REPO / "profiles" / args.round
    dst.mkdir(parents=True, exist_ok=True)
    for a, b in (("bench.json", "bench_N1.json"), ("bench_reference.json", "bench_reference_port.json")):
        line = (src / a).read_text().strip().splitlines()[-1]
        json.loads(line)
        (dst / b).write_text(line + "\n")
    for f in ("launches_bench.csv", "scan_stats.txt", "scan_timing.txt", "cycle_parts_config2.txt",
              "e2e_breakdown_config2.txt", "vmajor_config2.json", "vmajor_config5.json", "config3_precompute.json",
              "pytest_gpu.log", "placement_launches.csv"):
        if (src / f).exists():
            shutil.copy(src / f, dst / f)
    lines = [f"# ncu summaries, round {args.round[1:]} (tools/refresh_profiles.sh; B200, --clock-control none)", ""]
    lines += ["## launch list of the bench command (cold, serialised: shares, not absolutes)",
              _run([str(REPO / "tools" / "ncu_launches.py"), str(src / "launches_bench.csv")])]
    for w in ("config4", "config2"):
        rep = src / f"shells_{w}.ncu-rep"
        lines += [f"## query_shells_kernel, {w} (ncu --set full, the 4th cycle of bench.py --probe-counters)",
                  _run([str(REPO / "tools" / "ncu_summary.py"), str(rep)]),
                  "### hottest source lines", _run([str(REPO / "tools" / "ncu_lines.py"), str(rep), "30"])]
    if (src / "placement_launches.csv").exists():
        lines += ["## neural placement at config-3 scale (500 x 6 windows, W = 128): fused lsdf_mlp_place vs "
                  "TinyMlp + place_windows_g, and the exact place_windows (ncu, serialised)",
                  _run([str(REPO / "tools" / "ncu_launches.py"), str(src / "placement_launches.csv")])]
    rep = src / "cycle_config2.ncu-rep"
    lines += ["## every kernel of one config-2 cycle (ncu --set full)", _run([str(REPO / "tools" / "ncu_summary.py"),
                                                                            str(rep)])]
    (dst / "ncu_summary.txt").write_text("\n".join(lines))
    print("wrote", dst)


if __name__ == "__main__":
    main()
