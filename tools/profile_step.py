"""Run a few device-only steps of one workload for ncu (no CPU baseline, no timing).

    python tools/profile_step.py --workload config2 --steps 3
"""

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config2", choices=["config1", "config2", "config4"])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--device-only", action="store_true", help="inputs staged in HBM (the bench's value path)")
    ap.add_argument("--flush", action="store_true", help="write 256 MiB (evicts L2) before every step")
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
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(shape.n_waypoints, shape.n_points, np.float32,
                                                                use_graph=not args.no_graph)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    pts = S.cloud_for(shape, 11).astype(np.float32)
    if args.device_only:
        chk.q_dev.copy_(torch.from_numpy(q).cuda())
        chk.p_dev.copy_(torch.from_numpy(pts).cuda())
        junk = torch.empty(64 << 20, dtype=torch.float32, device="cuda") if args.flush else None
        for _ in range(args.steps):
            if junk is not None:
                junk.fill_(1.0)
            chk.launch(device_only=True)
        torch.cuda.synchronize()
        d, link = chk.d_dev.cpu().numpy(), chk.link_dev.cpu().numpy()
    else:
        for _ in range(args.steps):
            d, link, voxel = chk.query(q, pts)
    torch.cuda.synchronize()
    print("min d", float(d.min()), "links hit", int((link >= 0).sum()))


if __name__ == "__main__":
    main()
