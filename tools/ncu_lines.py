"""Per-source-line instruction and stall-sample shares of one ncu report (first kernel).

    python tools/ncu_lines.py report.ncu-rep [top] [kernel-regex]
"""
import csv
import subprocess
import sys


def main(path, top=30, kernel=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["--kernel-name", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    cur, hdr, rows = None, None, []
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0] not in ("", "Function Name") and len(r) > 7 and r[2] == "-":
            try:
                rows.append((int(float(r[7] or 0)), int(r[4] or 0), cur, r[0], r[1][:84]))
            except ValueError:
                pass
    ti = sum(x[0] for x in rows) or 1
    ts = sum(x[1] for x in rows) or 1
    print(f"warp instructions {ti}  stall samples {ts}")
    for x in sorted(rows, reverse=True)[:top]:
        print(f"inst {x[0] / ti:6.1%} samp {x[1] / ts:6.1%} {x[2]}:{x[3]} {x[4]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else None)
