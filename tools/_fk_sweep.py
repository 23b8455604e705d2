import sys, statistics, ctypes
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2309_12543_b200 as L
from paper_2309_12543_b200 import _native as N
from paper_2309_12543_b200 import scenarios as S
from paper_2309_12543_b200.robot import fk_device
robot = L.RobotModel.from_dict(S.ARM7G)
grid = L.EnvGrid(1.0, 0.04)
for C in (500, 2048, 4096, 8192, 16384, 32768, 65536):
    q = torch.from_numpy(S.random_configs(S.ARM7G, C, seed=1)).cuda()
    out = fk_device(robot, q, all_links=False, grid=grid, window_dims=[16, 16, 16])
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(10):
            fk_device(robot, q, all_links=False, grid=grid, window_dims=[16, 16, 16], outputs=out)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 100)  # us per launch
    print(C, round(statistics.median(ts), 1))
