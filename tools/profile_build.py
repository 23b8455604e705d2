"""Config-3 link-SDF builds for ncu: the six arm6g primitives and the 1,280-triangle icosphere at 128^3.

    python tools/profile_build.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    robot = L.RobotModel.from_dict(S.ARM6G)
    for i in robot.geometry_links:
        L.build_link_sdf(robot.links[i].geometry, 0.64, 0.01, link_id=i)
    ico = L.make_icosphere(0.08, subdivisions=3)
    sdf = L.build_link_sdf(ico, 0.64, 0.01)
    torch.cuda.synchronize()
    print("mesh grid min", float(sdf.device_values().min()))


if __name__ == "__main__":
    main()
