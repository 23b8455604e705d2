"""Host-side costs of one config-2 cycle: graph replay call, stream sync wait, result copies."""
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
    q_host, p_host = chk.host_inputs()
    q_host[...] = S.random_configs(shape.robot, shape.n_waypoints, seed=21)
    p = bench._cloud(shape, 21)
    p_host[: len(p)] = p
    g = chk._graph
    s = torch.cuda.current_stream()
    rep, syn, tot = [], [], []
    for k in range(300):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.replay()
        t1 = time.perf_counter()
        s.synchronize()
        t2 = time.perf_counter()
        chk.query()
        t3 = time.perf_counter()
        if k >= 20:
            rep.append(1e6 * (t1 - t0)); syn.append(1e6 * (t2 - t0)); tot.append(1e6 * (t3 - t2))
    raw = getattr(g, "raw_cuda_graph_exec", None)
    print(f"replay() call {np.median(rep):.1f} us; replay+sync {np.median(syn):.1f} us; query() {np.median(tot):.1f} us; "
          f"raw exec available: {raw is not None}")


if __name__ == "__main__":
    main()
