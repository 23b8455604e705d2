"""Device timeline of CheckerPipeline cycles (config 4): H2D, compute and D2H spans per cycle."""
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

    shape = bench._shape("config4")
    robot, chk = bench._checker(shape, shape.n_waypoints, L)
    depth = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    pipe = L.CheckerPipeline(robot, chk.sdfs, chk.grid, chk.window, shape.n_waypoints, shape.n_points, np.float32,
                             depth=depth)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    p = bench._cloud(shape, 11)
    for s in pipe.slots:
        qv, pv = s["chk"].host_inputs()
        qv[...], pv[...] = q, p
    # timing events around each piece (recorded on the pipeline's own streams)
    marks = []
    orig_launch = {}
    for k in range(8):
        pipe.result(pipe.submit())
    torch.cuda.synchronize()
    T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t0 = T()
    t0.record(pipe.compute)
    n = 40
    tickets = []
    ev = []
    w0 = time.perf_counter()
    for k in range(n):
        e = {x: T() for x in ("h2d0", "h2d1", "c0", "c1", "d0", "d1")}
        s = pipe._slot(pipe._next)
        if s["busy"]:
            pipe.result(s["ticket"])
        e["h2d0"].record(pipe.copy)
        ticket = pipe.submit()
        # submit enqueued copy -> compute -> d2h; bracket them after the fact on each stream
        e["h2d1"].record(pipe.copy)
        e["c1"].record(pipe.compute)
        e["d1"].record(pipe.d2h)
        ev.append(e)
        tickets.append(ticket)
    for t_ in tickets[-depth:]:
        pipe.result(t_)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    print(f"depth {depth}: host wall {1e3 * (w1 - w0) / n:.3f} ms/cycle")
    ends_c = [t0.elapsed_time(e["c1"]) for e in ev]
    ends_h = [t0.elapsed_time(e["h2d1"]) for e in ev]
    starts_h = [t0.elapsed_time(e["h2d0"]) for e in ev]
    ends_d = [t0.elapsed_time(e["d1"]) for e in ev]
    for k in range(5, 12):
        print(f"cycle {k}: h2d {starts_h[k]:8.3f} -> {ends_h[k]:8.3f} ({ends_h[k] - starts_h[k]:.3f})  compute end "
              f"{ends_c[k]:8.3f} (+{ends_c[k] - ends_c[k - 1]:.3f})  d2h end {ends_d[k]:8.3f}")
    print("median compute period", float(np.median(np.diff(ends_c[5:]))), "ms")


if __name__ == "__main__":
    main()
