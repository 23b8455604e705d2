"""Scan statistics from the instrumented build (-DLSDF_STATS): per-task chunks, occupied cells, lookups.

    python tools/scan_stats.py build          # here: builds _ab/libS.so
    python tools/scan_stats.py config4 ...    # on the GPU box
"""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
LIBS = REPO / "_ab" / "libS.so"


def build():
    from paper_2309_12543_b200 import build as B

    out = REPO / "_ab" / "stats"
    out.mkdir(parents=True, exist_ok=True)
    objs = []
    for name in B.SOURCES:
        obj = out / (Path(name).stem + ".o")
        subprocess.run([B._nvcc(), *B.ARCH, *B.FLAGS, "-DLSDF_STATS", "-I",
                        str(B.INCLUDE), "-c", str(B.CSRC / name), "-o", str(obj)], check=True, capture_output=True)
        objs.append(str(obj))
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(LIBS), *objs, "-lcuda"], check=True)
    print("built", LIBS)


def run(workload):
    os.environ["LINKSDF_B200_LIB"] = str(LIBS)
    import numpy as np
    import torch

    import bench
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import _native as N
    from paper_2309_12543_b200 import scenarios as S

    shape = bench._shape(workload)
    robot, chk = bench._checker(shape, shape.n_waypoints, L)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    chk.q_dev.copy_(torch.from_numpy(q).cuda())
    chk.p_dev.copy_(torch.from_numpy(bench._cloud(shape, 11)).cuda())
    lib = N.lib()
    f = lib.lsdf_stats_read
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 8)()
    for _ in range(3):
        chk.launch(device_only=True)
    torch.cuda.synchronize()
    f(buf, 1)
    chk.launch(device_only=True)
    torch.cuda.synchronize()
    f(buf, 1)
    s = np.array(list(buf), dtype=np.float64)
    n = s[0]
    print(f"{workload}: tasks {int(n)}  per task: chunks {s[1] / n:.2f}  chunks with occupancy {s[2] / n:.2f}  "
          f"occupied cells {s[3] / n:.1f}  queued (after segment bound) {s[4] / n:.1f}  lookup rounds "
          f"{s[5] / n:.2f}  early stops {s[6] / n:.3f}  stopped before any chunk {s[7] / n:.3f}")


if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:
        build()
    else:
        for w in sys.argv[1:]:
            run(w)
