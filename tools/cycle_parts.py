"""Device time of sub-graphs of the real-time cycle (which piece is on the critical path).

    python tools/cycle_parts.py [--workload config2] [--n 300] [--flush]

Every sub-graph is replayed behind a GPU spin (the host has enqueued it before
the start event fires), so each number is device execution, not launch latency.
"""
import argparse
import ctypes
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config2", choices=["config1", "config2", "config4"])
    ap.add_argument("--n", type=int, default=300)
    ap.add_argument("--flush", action="store_true")
    args = ap.parse_args()
    import torch

    import bench
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import _native as N
    from paper_2309_12543_b200 import scenarios as S

    shape = bench._shape(args.workload)
    robot, chk = bench._checker(shape, shape.n_waypoints, L)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=21)
    pts = bench._cloud(shape, 21)
    chk.q_dev.copy_(torch.from_numpy(q).cuda())
    chk.p_dev.copy_(torch.from_numpy(pts).cuda())
    C_, P, _ = chk._shape
    env = ctypes.byref(chk.grid.c_struct())
    tr = chk.traj
    cur = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    qargs = lambda: (N.ptr(chk.R_geo), N.ptr(chk.dt_geo), N.ptr(chk.anchor_geo), C_, tr.n_links, tr._table,  # noqa: E731
                     ctypes.byref(chk._wstruct), env, N.ptr(chk.ws), chk._qflags, chk.d_far_global, N.ptr(chk.qws),
                     N.ptr(chk.d_dev), N.ptr(chk.link_dev), N.ptr(chk.voxel_dev), None, cur())
    parts = {
        "fk": lambda: N.call(chk._fk_entry, chk._chain, robot.n_links, len(chk.sdfs), N.ptr(chk.q_dev), C_, robot.dof,
                             N.ptr(chk.limits), env, chk._W, None, None, N.ptr(chk.R_geo), N.ptr(chk.dt_geo),
                             N.ptr(chk.anchor_geo), N.ptr(chk.flags), cur()),
        "voxelize_bitmap": lambda: N.call("lsdf_voxelize_bitmap", N.ptr(chk.p_dev), 1, P, env, N.ptr(chk.ws), cur()),
        "prefix": lambda: N.call("lsdf_occupancy_prefix", env, N.ptr(chk.ws), cur()),
        "scan": lambda: N.call("lsdf_query_scan", *qargs()),
        "finalize": lambda: N.call("lsdf_query_finalize", *qargs()),
    }
    combos = {k: [k] for k in parts}
    combos["scan+finalize"] = ["scan", "finalize"]
    combos["vox+prefix+scan+finalize (serial)"] = ["voxelize_bitmap", "prefix", "scan", "finalize"]
    for f in parts.values():
        f()
    torch.cuda.synchronize()
    flush = bench.L2Flush(torch) if args.flush else (lambda: None)
    res = {}
    s = torch.cuda.Stream()
    for name, keys in combos.items():
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            for k in keys:
                parts[k]()
        torch.cuda.synchronize()
        ts = bench._time_steps(torch, g.replay, 20, flush)
        ts = bench._time_steps(torch, g.replay, args.n, flush)
        res[name] = statistics.median(ts) * 1e3
    ts = bench._time_steps(torch, lambda: chk.launch(device_only=True), args.n, flush)
    res["checker cycle graph"] = statistics.median(ts) * 1e3
    res["checker cycle graph mean"] = statistics.mean(ts) * 1e3
    res["checker cycle graph p99"] = float(np.percentile(ts, 99)) * 1e3
    print(json.dumps({"workload": args.workload, "flush": args.flush, "us": res}))
    for k, v in res.items():
        print(f"{k:40s} {v:8.1f} us")


if __name__ == "__main__":
    main()
