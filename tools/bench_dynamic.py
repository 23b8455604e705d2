"""BASELINE config 5 — dynamic scene: 100 control cycles of 8 ms re-querying a
500-waypoint trajectory against a human walking toward the robot.

    python tools/bench_dynamic.py [--check]

Per cycle: the frame's 30k points (f32) and the 500 configurations are read
from pinned host memory by the kernels, the cycle runs as one CUDA graph and
(d, link, voxel) land back in pinned memory.  Reports host-to-host and device
latency percentiles over the 100 frames, the number of frames whose closest
obstacle is inside the monitored range, and (--check) agreement with the
oracle port of the reference on every 10th frame.
"""

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--repeats", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG5
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    frames = S.moving_human_frames(100, shape.n_points, seed=5)
    q = S.smooth_trajectory(shape.robot, shape.n_waypoints, seed=5)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(shape.n_waypoints, shape.n_points, np.float32)
    q_host, p_host = chk.host_inputs()
    q_host[...] = q
    f32 = [(t, np.ascontiguousarray(p, dtype=np.float32)) for t, p in frames]
    for _ in range(10):
        p_host[...] = f32[0][1]
        chk.query()
    wall, results = [], []
    for rep in range(args.repeats):
        for t, p in f32:
            p_host[...] = p  # the sensor driver's write into the pinned frame buffer (not timed)
            t0 = time.perf_counter()
            d, link, voxel = chk.query()
            wall.append((time.perf_counter() - t0) * 1e6)
            if rep == 0:
                results.append((d, link, voxel))
    dev = []
    stream = torch.cuda.current_stream()
    for t, p in f32:
        chk.p_dev.copy_(torch.from_numpy(p).cuda())
        chk.q_dev.copy_(torch.from_numpy(q).cuda())
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        chk.launch(device_only=True)
        b.record(stream)
        b.synchronize()
        dev.append(a.elapsed_time(b) * 1e3)
    # the paper's two-phase mode: prepare the fixed trajectory's field once,
    # then one gather per cycle (MaterializedChecker)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mat = L.MaterializedChecker(robot, sdfs, grid, window, q)
    e1.record()
    e1.synchronize()
    prep_ms = e0.elapsed_time(e1)
    mat.prepare(shape.n_points, np.float32)
    mp = mat.host_points()
    for _ in range(10):
        mp[...] = f32[0][1]
        mat.query()
    wall_m, same = [], True
    for rep in range(args.repeats):
        for k, (t, p) in enumerate(f32):
            mp[...] = p
            t0 = time.perf_counter()
            dm, lm, vm = mat.query()
            wall_m.append((time.perf_counter() - t0) * 1e6)
            if rep == 0:
                same &= all(np.array_equal(a, b) for a, b in zip((dm, lm, vm), results[k]))
    near = sum(int((r[1] >= 0).any()) for r in results)
    out = {"config": "config5_dynamic", "frames": len(frames), "waypoints": shape.n_waypoints,
           "points_per_frame": shape.n_points, "cycle_budget_ms": 8.0,
           "e2e_p50_us": float(np.percentile(wall, 50)), "e2e_p99_us": float(np.percentile(wall, 99)),
           "e2e_max_us": float(np.max(wall)),
           "device_p50_us": float(np.percentile(dev, 50)), "device_p99_us": float(np.percentile(dev, 99)),
           "frames_with_obstacle_in_range": near,
           "min_distance_first_last": [float(results[0][0].min()), float(results[-1][0].min())],
           "zero_copy": chk.zero_copy,
           "materialized": {"prepare_ms_once": prep_ms, "e2e_p50_us": float(np.percentile(wall_m, 50)),
                            "e2e_p99_us": float(np.percentile(wall_m, 99)), "e2e_max_us": float(np.max(wall_m)),
                            "same_results_as_direct": bool(same),
                            "path": "MaterializedChecker: FK + exact placement + min-merge into a voxel-major "
                                    "(V, C) field once; per cycle one graph: zero-copy voxelize + gather + "
                                    "argmin-link pass"}}
    if args.check:
        from oracle import linksdf_oracle as O

        grids = [s.values for s in sdfs]
        bad = 0
        for k in range(0, len(frames), 10):
            rd, rl, rv = O.run_pipeline(shape.robot, q[::25], frames[k][1].astype(np.float32), shape.grid_extent,
                                        shape.grid_res, shape.link_extent, grids, [shape.link_res] * len(grids))
            d, link, voxel = results[k]
            ok = (np.abs(d[::25].astype(np.float64) - rd).max() <= 1e-6 and np.array_equal(link[::25], rl)
                  and np.array_equal(voxel[::25], rv))
            bad += not ok
        out["oracle_check"] = f"{10 - bad}/10 frames match (every 25th waypoint, d <= 1e-6 m, argmin exact)"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
