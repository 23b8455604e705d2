"""Where the host-to-host time of one control cycle goes (config 2 shape).

    python tools/e2e_breakdown.py [--workload config2] [--n 200]

Prints device time of the compute-only graph, of the full graph (with the
H2D/D2H copies), the bare H2D copy of the inputs, and the host wall clock of
DistanceChecker.query() — medians over n cycles.
"""

import argparse
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config2", choices=["config1", "config2", "config4"])
    ap.add_argument("--n", type=int, default=200)
    args = ap.parse_args()
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    shape = {"config1": S.CONFIG1, "config2": S.CONFIG2, "config4": S.CONFIG4}[args.workload]
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(shape.n_waypoints, shape.n_points, np.float32)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    pts = S.cloud_for(shape, 11).astype(np.float32)
    qh, ph = chk.host_inputs()
    qh[...] = q
    ph[: len(pts)] = pts
    stream = torch.cuda.current_stream()

    def dev_time(fn, n):
        out = []
        for _ in range(n):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            out.append(a.elapsed_time(b) * 1e3)
        return statistics.median(out)

    for _ in range(20):
        chk.query()
    res = {
        "compute_graph_us": dev_time(lambda: chk.launch(device_only=True), args.n),
        "full_graph_us": dev_time(lambda: chk.launch(), args.n),
        "h2d_points_us": dev_time(lambda: chk.p_dev.copy_(chk.p_host, non_blocking=True), args.n),
        "h2d_configs_us": dev_time(lambda: chk.q_dev.copy_(chk.q_host, non_blocking=True), args.n),
    }
    wall = []
    for _ in range(args.n):
        t0 = time.perf_counter()
        chk.query()
        wall.append((time.perf_counter() - t0) * 1e6)
    res["query_wall_us"] = statistics.median(wall)
    wall = []
    for _ in range(args.n):
        t0 = time.perf_counter()
        chk.launch()
        stream.synchronize()
        wall.append((time.perf_counter() - t0) * 1e6)
    res["launch_sync_wall_us"] = statistics.median(wall)
    wall = []
    for _ in range(args.n):
        t0 = time.perf_counter()
        chk.launch(device_only=True)
        stream.synchronize()
        wall.append((time.perf_counter() - t0) * 1e6)
    res["compute_launch_sync_wall_us"] = statistics.median(wall)
    for k, v in res.items():
        print(f"{k:30s} {v:9.1f}")


if __name__ == "__main__":
    main()
