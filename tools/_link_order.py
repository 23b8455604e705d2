"""EXPERIMENT: argmin-link histogram and scan time per link processing order (LSDF_GROUP_ORDER)."""
import os
import statistics
import subprocess
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def run(workload):
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
    link = chk.link_dev.cpu().numpy()
    d = chk.d_dev.cpu().numpy()
    flush = bench.L2Flush(torch)
    outs = {}
    qk = lambda: chk.traj.query_device(chk.ws, False, outputs=outs)  # noqa: E731
    bench._time_steps(torch, qk, 3, flush)
    t = bench._time_steps(torch, qk, 20, flush)
    h = np.bincount(link[link >= 0], minlength=len(chk.sdfs))
    print(f"{workload} order={os.environ.get('LSDF_GROUP_ORDER', 'default')} scan {1e3 * statistics.mean(t):.1f} us "
          f"argmin-link hist {h.tolist()} none {(link < 0).sum()} dsum {float(d.astype(np.float64).sum()):.6f}")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1])
    else:
        for w, n in (("config2", 6), ("config4", 7)):
            for order in ("", "".join(str(i) for i in reversed(range(n)))):
                env = dict(os.environ)
                if order:
                    env["LSDF_GROUP_ORDER"] = order
                subprocess.run([sys.executable, __file__, w], env=env)
