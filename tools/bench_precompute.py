"""BASELINE config 3 — per-link precompute at 128^3 and the grid transform at W = 128.

    python tools/bench_precompute.py [--cpu]

(i)   exact link-SDF build at 128^3 (e_r 0.64, r_r 0.01) for the six arm6g
      primitives and one 1,280-triangle mesh (icosphere, 3 subdivisions);
(ii)  exact grid transform G = P R + dt_inv (fp64, placement.py:148-169) for
      B = 3,000 rotations x V_mask = 1,097,911 cells (W = 128, r_e = 0.01);
(iii) TinyMlp prediction of the same G (approx.py:123-130) on tcgen05 tensor
      cores (3xTF32) and on CUDA cores.
Prints one JSON object: device times (CUDA events), achieved bandwidth/flops
and their roofline fractions, and (with --cpu) the oracle port timed on a
bounded, extrapolated sample.
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


def _time(torch, fn, reps=5, warm=3):
    """Median device time (ms); several warm-ups so the SM clock has ramped up from idle first."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--rotations", type=int, default=3000)
    ap.add_argument("--chunk", type=int, default=1000, help="rotations per exact-transform launch (fp64 G)")
    ap.add_argument("--mlp-chunk", type=int, default=3000, help="rotations per MLP launch (f32 y)")
    ap.add_argument("--train", action="store_true", help="train a W=128 model first and time that one")
    ap.add_argument("--placement", action="store_true", help="also time exact vs neural placement of 500 x 6 windows")
    ap.add_argument("--train-steps", type=int, default=40_000)
    args = ap.parse_args()
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import _native as N
    from paper_2309_12543_b200 import scenarios as S

    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tf32_peak = float(peaks.get("bf16_tflops", 1590.0)) / 2.0  # dense TF32 = bf16 / 2 (B200_PROFILING.md)
    out = {"config": "config3_precompute"}

    # (i) builds
    robot = L.RobotModel.from_dict(S.ARM6G)
    e_r, r_r = 0.64, 0.01
    builds, kernel_us = {}, {}
    from paper_2309_12543_b200.meshes import _primitive_params

    vals = torch.empty((128, 128, 128), dtype=torch.float32, device="cuda")
    for i in robot.geometry_links:
        g = robot.links[i].geometry
        ms = _time(torch, lambda: L.build_link_sdf(g, e_r, r_r, link_id=i))
        builds[robot.links[i].name] = ms
        kind, prm = _primitive_params(g)
        # the kernel alone: 20 launches through the C ABI captured in a CUDA graph (no host overhead)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            for _ in range(20):
                N.call("lsdf_build_primitive", kind, prm, N.f64s([e_r] * 3, 3), N.f64s([r_r] * 3, 3),
                       N.i32x3([128] * 3), N.ptr(vals), s.cuda_stream)
        kernel_us[robot.links[i].name] = 1e3 / 20 * _time(torch, g.replay)
    ico = L.make_icosphere(0.08, subdivisions=3)
    assert len(ico.triangles) == 1280
    ms_mesh = _time(torch, lambda: L.build_link_sdf(ico, e_r, r_r), reps=5)
    cells = 128 ** 3
    prim_ms = statistics.mean(builds.values())
    k_us = statistics.mean(kernel_us.values())
    out["build"] = {
        "primitive_ms_per_link": builds, "cells": cells,
        "primitive_kernel_us_per_link": kernel_us,
        "primitive_kernel_write_GBps": 4 * cells / (k_us / 1e6) / 1e9,
        "primitive_kernel_frac_hbm": 4 * cells / (k_us / 1e6) / 1e9 / hbm,
        "primitive_api_write_GBps": 4 * cells / (prim_ms / 1e3) / 1e9,
        "mesh_ms": ms_mesh, "mesh_triangles": 1280,
        "mesh_pairs_per_s": cells * 1280 / (ms_mesh / 1e3),
        "mesh_fp64_flop_per_s": 110.0 * cells * 1280 / (ms_mesh / 1e3),
        "mesh_note": "pairs/s and flop/s are algorithmic (every cell x every triangle, ~110 fp64 flop per pair, "
                     "as the reference computes); the kernel culls pairs that provably cannot change a result",
    }

    # (ii)/(iii) transform at W = 128
    grid = L.EnvGrid(1.28, 0.01)
    window = L.WindowGeometry.build(0.64, grid)
    V = window.n_masked
    rng = np.random.default_rng(0)
    B, ch = args.rotations, args.chunk
    Rall = L.sample_rotations(rng, B)
    dt = rng.uniform(-0.005, 0.005, size=(B, 3))
    P = N.to_device(window.masked_points, torch.float64)
    Rd = torch.from_numpy(Rall.reshape(B, 9)).cuda()
    dtd = torch.from_numpy(dt).cuda()
    G = torch.empty((ch, V, 3), dtype=torch.float64, device="cuda")

    def exact_all():
        for s in range(0, B, ch):
            N.call("lsdf_grid_transform_exact", N.ptr(Rd[s:s + ch]), N.ptr(dtd[s:s + ch]), ch, N.ptr(P), V, 0.64,
                   N.ptr(G), N.stream())

    ms_exact = _time(torch, exact_all, reps=5)
    del G
    training = None
    if args.train:
        # a real W = 128 model, trained here on the GPU (lsdf_train.cu; rotations
        # drawn on the device), used for the MLP timing and its accuracy check
        cfg = L.TrainingConfig(steps=args.train_steps, device_rng=True, val_size=2000)
        t0 = time.perf_counter()
        try:
            model = L.train_approximator(window.masked_points, cfg)
            converged = True
        except L.NotConvergedError as exc:
            model, converged = exc.model, False
        training = {"converged": converged, "steps": model.steps_run, "seconds": time.perf_counter() - t0,
                    "val_max_abs_error": model.validation_max_error,
                    "val_mean_abs_error": model.validation_mean_error, "target_max_error": cfg.target_max_error,
                    "history_tail": model.history[-3:],
                    "note": "TrainingConfig defaults (hidden 32, batch 64, lr 1e-4, L1 + Adam, stop at half the target "
                            "on the validation set), device-drawn rotations; 2,000 validation rotations"}
        out["training"] = training
    else:
        model = L.TinyMlp.initial(V, hidden=32, seed=0)
        model.w2 = np.random.default_rng(1).normal(0, 0.05, size=model.w2.shape).astype(np.float32)
        model._dev = None
    mch = args.mlp_chunk
    # rows at a 32-float stride (128-B aligned, the layout predict_device allocates)
    Y = torch.empty((mch, (3 * V + 31) // 32 * 32), dtype=torch.float32, device="cuda")[:, :3 * V]

    def mlp_all(tc):
        for s in range(0, B, mch):
            model.predict_device(Rd[s:s + mch], use_tensor_cores=tc, out=Y)

    ms_tc = _time(torch, lambda: mlp_all(True), reps=5)
    ms_cc = _time(torch, lambda: mlp_all(False), reps=5)
    flops = 2.0 * B * (9 * 32 + 32 * 3 * V)
    out["transform"] = {
        "rotations": B, "V_mask": V, "W": int(window.dims[0]), "chunk_exact": ch, "chunk_mlp": mch,
        "exact_fp64_ms": ms_exact, "exact_write_GBps": B * V * 24 / (ms_exact / 1e3) / 1e9,
        "exact_frac_hbm": B * V * 24 / (ms_exact / 1e3) / 1e9 / hbm,
        "mlp_tcgen05_ms": ms_tc, "mlp_cuda_core_ms": ms_cc,
        "mlp_algorithmic_flop": flops,
        "mlp_tcgen05_TFLOPs": flops / (ms_tc / 1e3) / 1e12,
        "mlp_tcgen05_frac_tf32_dense": flops / (ms_tc / 1e3) / 1e12 / tf32_peak,
        "mlp_tcgen05_write_GBps": B * V * 12 / (ms_tc / 1e3) / 1e9,
        "mlp_tcgen05_frac_hbm_write": B * V * 12 / (ms_tc / 1e3) / 1e9 / hbm,
        "tf32_dense_peak_TFLOPs": tf32_peak,
        "weights": "trained W=128 model (see training)" if training else "random W2 (no trained model)",
        "note": "the MLP costs 32 MACs per output coordinate vs 3 for the exact product; with both writing G the "
                "MLP is output-write bound (12 B/point f32) and the exact transform writes 24 B/point (fp64)",
    }
    # (iv) placement of 500 waypoints x 6 links at this window (placement.py:267-313):
    # exact transform vs the (trained) TinyMlp provider, windows on the device
    if args.placement:
        from paper_2309_12543_b200.placement import place_windows_device

        del Y
        torch.cuda.empty_cache()
        sdfs = [L.build_link_sdf(robot.links[i].geometry, e_r, r_r, link_id=i) for i in robot.geometry_links]
        q = S.random_configs(S.ARM6G, 500, seed=3)
        poses = L.forward_kinematics_batch(robot, L.ConfigBatch(q))
        gl = robot.geometry_links
        Rg = torch.from_numpy(np.ascontiguousarray(poses.rotations[:, gl])).cuda()
        Tg = torch.from_numpy(np.ascontiguousarray(poses.translations[:, gl]).reshape(-1, 3)).cuda()
        from paper_2309_12543_b200.placement import _align_device

        _, dtg, _ = _align_device(Tg, grid, window.dims)
        dtg = dtg.reshape(500, len(gl), 3)
        prov_n = L.NeuralTransformProvider(model, window, fused=True)
        ms_place_exact = _time(torch, lambda: place_windows_device(sdfs, Rg, dtg, window), reps=3, warm=1)
        torch.cuda.empty_cache()
        ms_place_neural = _time(torch, lambda: place_windows_device(sdfs, Rg, dtg, window, prov_n), reps=3, warm=1)
        torch.cuda.empty_cache()
        prov_2k = L.NeuralTransformProvider(model, window, fused=False)
        ms_place_2k = _time(torch, lambda: place_windows_device(sdfs, Rg, dtg, window, prov_2k), reps=3, warm=1)
        torch.cuda.empty_cache()
        wa = place_windows_device(sdfs, Rg, dtg, window, prov_n)
        wb = place_windows_device(sdfs, Rg, dtg, window, prov_2k)
        same = bool(torch.equal(wa.view(torch.int32), wb.view(torch.int32)))
        del wa, wb
        torch.cuda.empty_cache()
        out["placement"] = {"waypoints": 500, "links": len(gl), "windows": 500 * len(gl),
                            "cells_per_window": int(window.n_cells), "kept_per_window": V,
                            "exact_ms": ms_place_exact, "neural_fused_ms": ms_place_neural,
                            "neural_two_kernel_ms": ms_place_2k,
                            "fused_equals_two_kernel": same,
                            "window_bytes_written": 500 * len(gl) * int(window.n_cells) * 4,
                            "note": "neural_fused = lsdf_mlp_place (TinyMlp layer 2 on tcgen05 with the sampler in "
                                    "its epilogue, G never in HBM; opt-in); neural_two_kernel (the provider's default) "
                                    "= TinyMlp on tcgen05 writing G (f32) + provider-coordinate sampler reading it "
                                    "back; exact = fused fp64 transform + sampler"}
    if args.cpu:
        from oracle import linksdf_oracle as O

        geo = [l for l in S.ARM6G["links"] if l.get("geometry")][0]["geometry"]
        t0 = time.perf_counter()
        O.build_grid(geo, e_r, r_r)
        cpu_prim = time.perf_counter() - t0
        axes = O.cell_centers(e_r, r_r)
        sub = np.stack(np.meshgrid(axes[0][::16], axes[1][::16], axes[2][::16], indexing="ij"), -1).reshape(-1, 3)
        t0 = time.perf_counter()
        O.mesh_sdf(ico.vertices, ico.triangles, sub, signed=True)
        cpu_mesh_s = (time.perf_counter() - t0) * cells / len(sub)
        pts = window.masked_points
        t0 = time.perf_counter()
        O.transform_exact(Rall[:2], dt[:2], 0.64, pts)
        cpu_exact_s = (time.perf_counter() - t0) / 2 * B
        t0 = time.perf_counter()
        O.mlp_predict(model.w1, model.b1, model.w2, model.b2, Rall[:2])
        cpu_mlp_s = (time.perf_counter() - t0) / 2 * B
        out["cpu_port"] = {"primitive_build_s": cpu_prim, "mesh_build_s_extrapolated": cpu_mesh_s,
                           "exact_transform_s_extrapolated": cpu_exact_s, "mlp_predict_s_extrapolated": cpu_mlp_s,
                           "sample": "oracle port (numpy, 1 process); mesh: every 16th cell per axis; transforms: "
                                     "2 rotations scaled to 3,000"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
