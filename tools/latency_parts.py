"""Graph-replay latency of sub-graphs of one cycle (which stage is on the critical path).

    python tools/latency_parts.py [--workload config2] [--n 300]
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
    ap.add_argument("--n", type=int, default=300)
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
    C_, P, _ = chk._shape
    env = ctypes.byref(grid.c_struct())
    s = torch.cuda.Stream()

    def fk():
        N.call(chk._fk_entry, chk._chain, robot.n_links, len(sdfs), N.ptr(chk.q_dev), C_, robot.dof,
               N.ptr(chk.limits), env, chk._W, None, None, N.ptr(chk.R_geo), N.ptr(chk.dt_geo), N.ptr(chk.anchor_geo),
               N.ptr(chk.flags), torch.cuda.current_stream().cuda_stream)

    def vox():
        N.call("lsdf_voxelize", N.ptr(chk.p_dev), 1, P, env, N.ptr(chk.ws), None,
               torch.cuda.current_stream().cuda_stream)

    def query():
        tr = chk.traj
        N.call("lsdf_query_direct", N.ptr(chk.R_geo), N.ptr(chk.dt_geo), N.ptr(chk.anchor_geo), C_, tr.n_links,
               tr._table, ctypes.byref(chk._wstruct), env, N.ptr(chk.ws), chk._qflags, chk.d_far_global, N.ptr(chk.qws),
               N.ptr(chk.d_dev), N.ptr(chk.link_dev), N.ptr(chk.voxel_dev), None,
               torch.cuda.current_stream().cuda_stream)

    def empty():
        pass

    parts = {"empty": [empty], "fk": [fk], "voxelize": [vox], "fk+voxelize(serial)": [fk, vox],
             "query": [query], "vox+query": [vox, query], "full(serial)": [fk, vox, query]}
    for fn in (fk, vox, query):
        fn()
    torch.cuda.synchronize()
    res = {}
    for name, fns in parts.items():
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for fn in fns:
                    fn()
        torch.cuda.synchronize()
        for _ in range(20):
            g.replay()
        ts = []
        for _ in range(args.n):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[name] = statistics.median(ts)
    ts = []
    for _ in range(args.n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        chk.launch(device_only=True)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    res["checker graph (fk || vox, query)"] = statistics.median(ts)
    for k, v in res.items():
        print(f"{k:36s} p50 {v:8.1f} us")


if __name__ == "__main__":
    main()
