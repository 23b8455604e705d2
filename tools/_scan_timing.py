"""A/B helper: scan (+finalize) and whole-cycle device times, L2 flushed vs warm, host launch hidden."""
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main(workload):
    import torch

    import bench
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    shape = bench._shape(workload)
    robot, chk = bench._checker(shape, shape.n_waypoints, L)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    chk.q_dev.copy_(torch.from_numpy(q).cuda())
    chk.p_dev.copy_(torch.from_numpy(bench._cloud(shape, 11)).cuda())
    chk.launch(device_only=True)
    torch.cuda.synchronize()
    flush = bench.L2Flush(torch)
    outs = {}
    qk = lambda: chk.traj.query_device(chk.ws, False, outputs=outs)  # noqa: E731
    cyc = lambda: chk.launch(device_only=True)  # noqa: E731
    nof = lambda: None  # noqa: E731
    for name, fn in (("scan", qk), ("cycle", cyc)):
        for fl, f in (("flushed", flush), ("warm", nof)):
            bench._time_steps(torch, fn, 5, f)
            t = bench._time_steps(torch, fn, 50, f)
            print(f"{workload} {name:5s} {fl:7s} mean {1e3 * statistics.mean(t):8.1f} us  p50 "
                  f"{1e3 * float(np.median(t)):8.1f} us")


if __name__ == "__main__":
    for w in sys.argv[1:] or ["config2", "config4"]:
        main(w)
