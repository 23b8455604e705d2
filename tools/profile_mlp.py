"""A few TinyMlp predictions at config-3 shape (W = 128, B = 3,000) for ncu.

    python tools/profile_mlp.py [--reps 3] [--cuda-core]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rotations", type=int, default=3000)
    ap.add_argument("--cuda-core", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import _native as N
    from paper_2309_12543_b200.approx import sample_rotations

    grid = L.EnvGrid(0.64, 0.01)
    window = L.WindowGeometry.build(0.64, grid)
    V = window.n_masked
    model = L.TinyMlp.initial(V, hidden=32, seed=0)
    model.w2 = np.random.default_rng(1).normal(0, 0.05, size=model.w2.shape).astype(np.float32)
    model._dev = None
    R = N.to_device(sample_rotations(np.random.default_rng(0), args.rotations).reshape(-1, 9), torch.float64)
    Y = torch.empty((args.rotations, (3 * V + 31) // 32 * 32), dtype=torch.float32, device="cuda")[:, :3 * V]
    for _ in range(args.reps):
        model.predict_device(R, use_tensor_cores=not args.cuda_core, out=Y)
    torch.cuda.synchronize()
    print("V", V, "y[0,:3]", Y[0, :3].tolist())


if __name__ == "__main__":
    main()
