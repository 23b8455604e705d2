"""Train a TinyMlp on the GPU (lsdf_train.cu) for a window width and save it (TMLP file).

    python tools/train_tmlp.py --width 128 --out gpurun_out/tmlp_w128.tmlp [--steps N] [--time-only]

Width 128 is BASELINE config 3's window (e_r 0.64 m, r_e 0.01 m: 1,097,911
kept cells, 3,293,733 outputs); the reference's defaults (hidden 32, batch 64,
lr 1e-4, L1 + Adam, early stop at half the 1.3e-3 target) with rotations drawn
on the device.  Prints one JSON summary (steps, ms per step, validation errors).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=128)
    ap.add_argument("--steps", type=int, default=200_000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--time-only", action="store_true", help="time 200 steps, no convergence run")
    ap.add_argument("--val-size", type=int, default=10_000)
    args = ap.parse_args()
    import torch

    import paper_2309_12543_b200 as L

    pts = L.masked_window_points(args.width)
    if args.time_only:
        cfg = L.TrainingConfig(steps=20, eval_every=10**9, screen_size=8, val_size=8, target_max_error=1e9,
                               device_rng=True)
        L.train_approximator(pts, cfg)  # warm-up
        torch.cuda.synchronize()
        cfg = L.TrainingConfig(steps=200, eval_every=10**9, screen_size=8, val_size=8, target_max_error=1e9,
                               device_rng=True)
        t0 = time.perf_counter()
        L.train_approximator(pts, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"width": args.width, "n_points": len(pts), "steps": 200, "ms_per_step": 1e3 * dt / 200}))
        return
    cfg = L.TrainingConfig(steps=args.steps, device_rng=True, val_size=args.val_size)
    t0 = time.perf_counter()
    try:
        model = L.train_approximator(pts, cfg)
        ok = True
    except L.NotConvergedError as exc:
        model, ok = exc.model, False
    dt = time.perf_counter() - t0
    if args.out:
        model.save(args.out)
    print(json.dumps({"width": args.width, "n_points": len(pts), "converged": ok, "steps": model.steps_run,
                      "seconds": dt, "ms_per_step": 1e3 * dt / max(1, model.steps_run),
                      "val_max_abs_error": model.validation_max_error, "val_mean_abs_error": model.validation_mean_error,
                      "target_max_error": cfg.target_max_error, "history": model.history[-5:]}))


if __name__ == "__main__":
    main()
