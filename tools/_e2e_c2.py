"""A/B helper: config-2 host-to-host cycle (DistanceChecker.query) p50/p99, L2 flushed before each."""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import bench
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    shape = bench._shape("config2")
    robot, chk = bench._checker(shape, shape.n_waypoints, L)
    inputs = [(S.random_configs(shape.robot, shape.n_waypoints, seed=s), bench._cloud(shape, s)) for s in (21, 22, 23, 24)]
    flush = bench.L2Flush(torch)
    q_host, p_host = chk.host_inputs()
    ts = []
    for k in range(300):
        q, p = inputs[k % 4]
        q_host[...] = q
        p_host[: len(p)] = p
        flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chk.query()
        if k >= 20:
            ts.append(1e6 * (time.perf_counter() - t0))
    print(f"e2e p50 {np.percentile(ts, 50):.1f} us  p99 {np.percentile(ts, 99):.1f} us")


if __name__ == "__main__":
    main()
