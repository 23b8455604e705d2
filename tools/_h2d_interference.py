"""Does a concurrent pinned H2D stream slow the config-4 cycle graph?  (device-only replays)"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import bench
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    shape = bench._shape("config4")
    robot, chk = bench._checker(shape, shape.n_waypoints, L)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    chk.q_dev.copy_(torch.from_numpy(q).cuda())
    chk.p_dev.copy_(torch.from_numpy(bench._cloud(shape, 11)).cuda())
    n = 16 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    for mode in ("alone", "with_h2d", "with_d2d", "alone"):
        ts = []
        for k in range(25):
            torch.cuda.synchronize()
            if mode == "with_h2d":
                with torch.cuda.stream(side):
                    for _ in range(3):
                        d.copy_(h, non_blocking=True)
            if mode == "with_d2d":
                with torch.cuda.stream(side):
                    for _ in range(3):
                        d[: chk.p_dev.numel() * 4].copy_(chk.p_dev.view(torch.uint8).reshape(-1), non_blocking=True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            chk.launch(device_only=True)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        print(f"{mode:9s} cycle p50 {statistics.median(ts[5:]):.1f} us")


if __name__ == "__main__":
    main()
