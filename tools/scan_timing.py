"""Where the shell scan's time goes on the latency path: globaltimer stamps per
warp / grab / task from an instrumented build (-DLSDF_TIMING).

    python tools/scan_timing.py build          # here: builds _ab/timing/liblinksdf_b200.so
    python tools/scan_timing.py config2 ...    # on the GPU box
"""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
LIBT = REPO / "_ab" / "timing" / "liblinksdf_b200.so"


def build():
    from paper_2309_12543_b200 import build as B

    out = LIBT.parent
    out.mkdir(parents=True, exist_ok=True)
    objs = []
    for name in B.SOURCES:
        obj = out / (Path(name).stem + ".o")
        subprocess.run([B._nvcc(), *B.ARCH, *B.FLAGS, "-DLSDF_TIMING", "-I", str(B.INCLUDE), "-c", str(B.CSRC / name),
                        "-o", str(obj)], check=True, capture_output=True)
        objs.append(str(obj))
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(LIBT), *objs, "-lcuda"], check=True)
    print("built", LIBT)


def run(workload):
    os.environ["LINKSDF_B200_LIB"] = str(LIBT)
    import numpy as np
    import torch

    import bench
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import _native as N
    from paper_2309_12543_b200 import scenarios as S

    shape = bench._shape(workload)
    robot, chk = bench._checker(shape, shape.n_waypoints, L)
    chk.q_dev.copy_(torch.from_numpy(S.random_configs(shape.robot, shape.n_waypoints, seed=21)).cuda())
    chk.p_dev.copy_(torch.from_numpy(bench._cloud(shape, 21)).cuda())
    f = N.lib().lsdf_timing_read
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 16)()
    flush = bench.L2Flush(torch)
    acc = np.zeros(16)
    reps = 50
    for k in range(reps + 3):
        flush()
        torch.cuda.synchronize()
        f(buf, 1)
        chk.launch(device_only=True)
        torch.cuda.synchronize()
        f(buf, 0)
        if k >= 3:
            acc += np.array(list(buf), dtype=np.float64)
    s = acc / reps
    warps, grabs, tasks = s[2], s[4], s[5]
    print(f"{workload}: per cycle {warps:.0f} warps, {grabs:.0f} later grabs, {tasks:.0f} later tasks")
    print(f"  kernel span (first warp entry -> last warp exit)  {(s[8] - s[0]) / 1e3:7.2f} us")
    print(f"  prologue per warp (entry -> tables staged, incl. first setup) {s[1] / warps / 1e3:7.2f} us")
    print(f"  warp lifetime mean {s[9] / warps / 1e3:7.2f} us, after staging {s[10] / warps / 1e3:7.2f} us")
    if grabs:
        print(f"  later grabs: setup {s[3] / grabs / 1e3:7.2f} us, scan {s[6] / grabs / 1e3:7.2f} us, "
              f"flush {s[7] / grabs / 1e3:7.2f} us per grab ({tasks / grabs:.1f} tasks)")


if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:
        build()
    else:
        for w in sys.argv[1:]:
            run(w)
