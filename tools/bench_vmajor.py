"""The paper's materialized mode (voxel-major field) vs the fused direct query.

    python tools/bench_vmajor.py [--workload config2|config5]

Prints one JSON object: the per-trajectory preparation (FK + exact placement +
min-merge into the (V, C) field), the per-cycle device time of the gather
query (voxelize with the sorted list + lsdf_query_vm, CUDA graph, L2 warm and
flushed), the same cycle through the fused direct query, and the gather
kernel's HBM roofline (4 B per (occupied voxel, configuration)).
"""
import argparse
import ctypes
import json
import statistics
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config2", choices=["config2", "config5"])
    ap.add_argument("--n", type=int, default=200)
    args = ap.parse_args()
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import _native as N
    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG2 if args.workload == "config2" else S.CONFIG5
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=21)
    pts = (S.cloud_for(shape, 21) if shape.cloud != "moving"
           else S.moving_human_frames(n_frames=100, seed=21)[60][1]).astype(np.float32)
    C_ = shape.n_waypoints

    def timed(fn, n, flush=None):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        out = []
        for _ in range(n):
            if flush is not None:
                flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            out.append(a.elapsed_time(b) * 1e3)  # us
        return out

    # preparation per trajectory (device)
    q_dev = torch.from_numpy(q).cuda()
    state = {}

    def prep():
        traj = L.TrajectorySdf.from_configs(robot, q_dev, sdfs, grid, window, check=False)
        state["traj"], state["vm"] = traj, traj.materialize()

    prep_us = timed(prep, 20)
    traj, vm = state["traj"], state["vm"]

    # one cycle: voxelize (with the sorted list) + gather query, as a CUDA graph
    p_dev = torch.from_numpy(pts).cuda()
    env = ctypes.byref(grid.c_struct())
    occ = L.query.occupancy_workspace(grid)
    idx = torch.empty((grid.n_voxels, 3), dtype=torch.int32, device="cuda")
    outs = {}

    def cycle_vm():
        N.call("lsdf_voxelize", N.ptr(p_dev), 1, len(pts), env, N.ptr(occ), N.ptr(idx), N.stream())
        vm.query_device(occ, idx, -1, outputs=outs)

    def query_only():
        vm.query_device(occ, idx, -1, outputs=outs)

    s = torch.cuda.Stream()
    graphs = {}
    for name, fn in (("cycle", cycle_vm), ("query", query_only)):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            fn()
        graphs[name] = g
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cyc = timed(graphs["cycle"].replay, args.n)
    cyc_cold = timed(graphs["cycle"].replay, args.n, flush=flush_buf.zero_)
    qk = timed(graphs["query"].replay, args.n)
    n_occ = int(occ[:4].view(torch.int32).item())
    # the direct path on the same inputs (checker graph, device-only)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(C_, len(pts), np.float32)
    chk.q_dev.copy_(q_dev)
    chk.p_dev.copy_(p_dev)
    direct = timed(lambda: chk.launch(device_only=True), args.n)
    torch.cuda.synchronize()
    d_vm, d_direct = outs["d"].cpu().numpy(), chk.d_dev.cpu().numpy()
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text())
    alg = 4.0 * n_occ * C_
    q50 = statistics.median(qk)
    out = {
        "workload": f"{shape.name}: {C_} waypoints, {len(pts)} points, {n_occ} occupied voxels, field "
                    f"{grid.n_voxels} x {C_} f32 ({grid.n_voxels * C_ * 4 / 2**20:.0f} MiB)",
        "prepare_per_trajectory_ms_p50": statistics.median(prep_us) / 1e3,
        "cycle_vm_us_p50": statistics.median(cyc), "cycle_vm_us_p99": float(np.percentile(cyc, 99)),
        "cycle_vm_l2_flushed_us_p50": statistics.median(cyc_cold),
        "cycle_direct_us_p50": statistics.median(direct),
        "query_vm_graph_us_p50": q50,
        "query_vm_algorithmic_GBps": alg / (q50 * 1e-6) / 1e9,
        "query_vm_frac_hbm": alg / (q50 * 1e-6) / 1e9 / float(peaks["hbm_gbs"]),
        "same_result_as_direct": bool(np.array_equal(d_vm, d_direct)),
        "paper_preparation_ms_per_trajectory": 0.391,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
