"""Warm per-stage device times of one cycle (CUDA events, medians), config 2 by default.

    python tools/stage_times.py [--workload config2] [--n 200] [--flush]
"""

import argparse
import ctypes
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config2", choices=["config1", "config2", "config4"])
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--flush", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import _native as N
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
    chk.q_dev.copy_(torch.from_numpy(q).cuda())
    chk.p_dev.copy_(torch.from_numpy(pts).cuda())
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    C_, P, _ = chk._shape
    env = ctypes.byref(grid.c_struct())

    def fk():
        N.call(chk._fk_entry, chk._chain, robot.n_links, len(sdfs), N.ptr(chk.q_dev), C_, robot.dof,
               N.ptr(chk.limits), env, chk._W, None, None, N.ptr(chk.R_geo), N.ptr(chk.dt_geo), N.ptr(chk.anchor_geo),
               N.ptr(chk.flags), N.stream())

    def vox():
        N.call("lsdf_voxelize", N.ptr(chk.p_dev), 1, P, env, N.ptr(chk.ws), None, N.stream())

    def query():
        tr = chk.traj
        N.call("lsdf_query_direct", N.ptr(chk.R_geo), N.ptr(chk.dt_geo), N.ptr(chk.anchor_geo), C_, tr.n_links,
               tr._table, ctypes.byref(chk._wstruct), env, N.ptr(chk.ws), chk._qflags, chk.d_far_global, N.ptr(chk.qws),
               N.ptr(chk.d_dev), N.ptr(chk.link_dev), N.ptr(chk.voxel_dev), None, N.stream())

    def graph():
        chk.launch(device_only=True)

    res = {}
    for name, fn in (("fk_align", fk), ("voxelize", vox), ("query", query), ("graph_cycle", graph)):
        for _ in range(10):
            fn()
        ts = []
        for _ in range(args.n):
            if args.flush:
                flush_buf.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[name] = (statistics.median(ts), float(np.percentile(ts, 99)))
    for k, (p50, p99) in res.items():
        print(f"{k:14s} p50 {p50:8.1f} us   p99 {p99:8.1f} us")


if __name__ == "__main__":
    main()
