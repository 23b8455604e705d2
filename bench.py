"""Benchmark of the batched link-SDF distance checker (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload config4|config2]

One JSON line on rank 0.  A *step* is one pass of the hot path over one batch:
FK + alignment for every waypoint, voxelization of the step's obstacle cloud,
and the fused transform/trilinear/min/argmin query, producing
(d, link, voxel) per waypoint.

* ``value`` — waypoint-queries/s, whole job, on BASELINE config 4 (7-DoF arm,
  65,536 waypoints vs a 1M-point crowd cloud, 64^3 link SDFs, W = 16), inputs
  resident in HBM, device time (CUDA events on the launching stream), L2
  flushed (256 MiB write) before every timed step.  N > 1 GPUs: waypoints are
  sharded contiguously across ranks (no collective on the data path), time is
  the max over ranks.
* ``realtime`` (N = 1) — BASELINE config 2: p50/p99 µs per 500-waypoint query
  (6-DoF, 100k-point cloud, 64^3), device-only graph and host-to-host e2e.
* ``e2e`` — the same throughput through the public API (DistanceChecker.query)
  from pinned host buffers, H2D of configs + cloud and D2H of results inside
  the timed region.
* ``roofline`` — query_direct_kernel: algorithmic bytes 4·N_occ per
  waypoint-query (the reference's gather) over its event-timed
  duration, against MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline`` — the oracle port of the reference pipeline (numpy) on the
  host cores, bounded sample, rank 0 at N = 1.

``--impl reference`` times that CPU port alone on the same workload and
prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "p50/p99 µs per 500-waypoint query; waypoint-queries/s at 1/2/4/8 B200"
KERNELS_PER_STEP = 4  # fk_align, voxel_scatter, voxel_compact, query_direct (+1 memset node)


def _peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- workloads


def _shape(name):
    from paper_2309_12543_b200 import scenarios as S

    return {"config4": S.CONFIG4, "config2": S.CONFIG2, "config1": S.CONFIG1}[name]


def _cloud(shape, seed):
    from paper_2309_12543_b200 import scenarios as S

    return S.cloud_for(shape, seed).astype(np.float32)  # frames are f32 on disk (query.py:313-327)


def _setup_gpu(shape, n_configs, seeds, L):
    from paper_2309_12543_b200 import scenarios as S

    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(n_configs, shape.n_points, np.float32)
    inputs = [(S.random_configs(shape.robot, n_configs, seed=s), _cloud(shape, s)) for s in seeds]
    return robot, grid, sdfs, window, chk, inputs


class L2Flush:
    def __init__(self, torch):
        self.buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def __call__(self):
        self.buf.zero_()


def _time_steps(torch, fn, steps, flush, before=None):
    """Per-step device times (ms) with CUDA events on the launching stream."""
    stream = torch.cuda.current_stream()
    times = []
    for k in range(steps):
        if before is not None:
            before(k)
        flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        times.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in times]


def run_ours(args, rank, world, dist):
    import torch

    import paper_2309_12543_b200 as L

    torch.cuda.set_device(_env_int("LOCAL_RANK", 0))
    shape = _shape(args.workload)
    C_total = shape.n_waypoints
    per = C_total // world
    lo = rank * per
    n_local = per if rank < world - 1 else C_total - lo
    from paper_2309_12543_b200 import scenarios as S

    seeds = [11, 12, 13]
    robot, grid, sdfs, window, chk, _ = _setup_gpu(shape, n_local, [], L)
    # shard: each rank owns waypoints [lo, lo + n_local) of every step's trajectory batch
    dev_inputs = []
    for s in seeds:
        q_all = S.random_configs(shape.robot, C_total, seed=s)[lo:lo + n_local]
        dev_inputs.append((torch.from_numpy(np.ascontiguousarray(q_all)).cuda(),
                           torch.from_numpy(_cloud(shape, s)).cuda()))
    flush = L2Flush(torch)

    def stage(k):
        q, p = dev_inputs[k % len(dev_inputs)]
        chk.q_dev.copy_(q)
        chk.p_dev.copy_(p)

    step = lambda: chk.launch(device_only=True)  # noqa: E731
    _time_steps(torch, step, args.warmup, flush, stage)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        dev_ms = _time_steps(torch, step, args.steps, flush, stage)
    torch.cuda.synchronize()
    total_ms = sum(dev_ms)
    if dist is not None:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    value = C_total / (ms_per_step / 1e3)

    # ---- e2e through the public API from pinned host buffers (host wall clock)
    q_host, p_host = chk.host_inputs()
    host_np = [(q.cpu().numpy(), p.cpu().numpy()) for q, p in dev_inputs]
    e2e_t = []
    for k in range(args.warmup + args.steps):
        q, p = host_np[k % len(host_np)]
        q_host[...] = q
        p_host[: len(p)] = p
        flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d, link, voxel = chk.query()
        t1 = time.perf_counter()
        if k >= args.warmup:
            e2e_t.append(t1 - t0)
    e2e_ms = 1e3 * sum(e2e_t) / len(e2e_t)
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- roofline of the dominant kernel (query_direct) timed alone
    stage(0)
    chk.launch(device_only=True)
    torch.cuda.synchronize()
    n_occ = int(chk.ws[:4].view(torch.int32).item())
    q_outs = {}
    qk = lambda: chk.traj.query_device(chk.ws, False, outputs=q_outs)  # noqa: E731
    _time_steps(torch, qk, 3, flush)
    q_ms = statistics.mean(_time_steps(torch, qk, max(5, args.steps), flush))
    alg_bytes = 4.0 * n_occ * n_local
    peak, peak_kind = _peaks()
    achieved = alg_bytes / (q_ms / 1e3) / 1e9
    traffic = None
    tf = REPO / "profiles" / "query_direct_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(args.workload)
        except (ValueError, OSError):
            traffic = None
    out = {
        "metric": METRIC, "value": value, "unit": "waypoint-queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 index math + f32 lerp",
        "data": "synthetic (seeded scenarios: arm7g/arm6g primitives, human/crowd clouds)",
        "config": {"workload": f"{shape.name}: {shape.robot['name']} {C_total} waypoints vs {shape.n_points} pts "
                               f"({shape.cloud}), link SDF {round(2 * shape.link_extent / shape.link_res)}^3, "
                               f"env 50^3 @ 4 cm, W=16", "waypoints": C_total, "points": shape.n_points,
                   "occupied_voxels": n_occ, "parallelism": f"waypoint shards x{world}",
                   "l2": "flushed (256 MiB write) before every timed step"},
        "gpu_launches": KERNELS_PER_STEP * args.steps,
        "e2e": {"value": C_total / (e2e_ms / 1e3), "unit": "waypoint-queries/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(n_local * robot.dof * 8 + shape.n_points * 12),
                "d2h_bytes_per_step": int(n_local * 12 + 16),
                "path": "DistanceChecker.query() from pinned host buffers, one CUDA graph, host wall clock"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "query_direct_kernel", "kernel_ms": q_ms,
                     "algorithmic_bytes": alg_bytes, "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
        "clocks": sampler.summary(),
    }
    return out, (robot, grid, sdfs, window, chk, n_occ)


def run_realtime(args, L):
    """Config 2: p50/p99 per 500-waypoint query (device graph and host-to-host)."""
    import torch

    shape = _shape("config2")
    seeds = [21, 22, 23, 24]
    robot, grid, sdfs, window, chk, inputs = _setup_gpu(shape, shape.n_waypoints, seeds, L)
    dev_inputs = [(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda()) for q, p in inputs]
    flush = L2Flush(torch)

    def stage(k):
        q, p = dev_inputs[k % len(dev_inputs)]
        chk.q_dev.copy_(q)
        chk.p_dev.copy_(p)

    n = max(50, args.steps)
    _time_steps(torch, lambda: chk.launch(device_only=True), 10, flush, stage)
    dev = _time_steps(torch, lambda: chk.launch(device_only=True), n, flush, stage)
    q_host, p_host = chk.host_inputs()
    e2e = []
    for k in range(n + 10):
        q, p = inputs[k % len(inputs)]
        q_host[...] = q
        p_host[: len(p)] = p
        flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chk.query()
        if k >= 10:
            e2e.append(1e3 * (time.perf_counter() - t0))
    chk.launch(device_only=True)
    torch.cuda.synchronize()
    n_occ = int(chk.ws[:4].view(torch.int32).item())
    pct = lambda a, p: float(np.percentile(np.asarray(a) * 1e3, p))  # noqa: E731  ms -> µs
    return {"workload": f"{shape.name}: arm6g 500 waypoints vs 100k pts, 64^3, W=16", "occupied_voxels": n_occ,
            "device_p50_us": pct(dev, 50), "device_p99_us": pct(dev, 99),
            "e2e_p50_us": pct(e2e, 50), "e2e_p99_us": pct(e2e, 99), "samples": n,
            "waypoint_queries_per_s_device": 500 / (statistics.mean(dev) / 1e3)}


# ----------------------------------------------------------------------------- CPU (oracle port)


def cpu_baseline(workload: str, budget_s: float = 20.0):
    """Time the oracle port (numpy restatement of the reference) on a bounded sample."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200 import scenarios as S

    shape = _shape(workload)
    doc = shape.robot
    chain = O.chain_from_doc(doc)
    gl = O.geometry_links(chain)
    grids = [O.build_grid(chain[i]["geometry"], shape.link_extent, shape.link_res) for i in gl]
    env = O.Env(shape.grid_extent, shape.grid_res)
    pts = _cloud(shape, 11)
    t0 = time.perf_counter()
    idx, _, _ = O.voxelize(pts, env)
    t_vox = time.perf_counter() - t0
    sample = 64 if workload == "config4" else shape.n_waypoints
    q = S.random_configs(doc, sample, seed=11)
    reps, t_run = 0, 0.0
    while reps < 2 or (t_run < budget_s and reps < 5):
        t0 = time.perf_counter()
        R, T = O.fk(chain, q)
        windows, anchors = O.place_windows(grids, [shape.link_extent] * len(gl), [shape.link_res] * len(gl),
                                           R[:, gl], T[:, gl], env, shape.link_extent)
        batch = O.assemble(windows, anchors, env, shape.link_extent)
        O.argmin_oracle(batch, windows, anchors, idx, shape.link_extent)
        t_run += time.perf_counter() - t0
        reps += 1
    t_sample = t_run / reps
    # per-waypoint rate with the cloud's voxelization charged pro rata (it runs
    # once per step for all waypoints of the step)
    t_per_wp = t_sample / sample + t_vox / shape.n_waypoints
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or "default"
    return {"value": 1.0 / t_per_wp, "unit": "waypoint-queries/s", "cores": len(os.sched_getaffinity(0)),
            "kind": "port",
            "sample": f"{shape.name}: {sample} waypoints x {reps} reps through FK+placement+assembly+gather+argmin "
                      f"({t_sample:.2f} s each) + voxelize of the full {shape.n_points}-pt cloud ({t_vox:.2f} s, "
                      f"charged per waypoint over {shape.n_waypoints}); numpy single process, "
                      f"OPENBLAS_NUM_THREADS={threads}",
            "seconds_per_waypoint": t_per_wp}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    shape = _shape(args.workload)
    samples = []
    base = None
    for k in range(args.warmup + args.steps):
        base = cpu_baseline(args.workload, budget_s=0.0)
        if k >= args.warmup:
            samples.append(base["value"])
        if sum(1 for _ in samples) and time.perf_counter() - _T0 > 240:
            break
    value = statistics.mean(samples) if samples else base["value"]
    return {"metric": METRIC, "value": value, "unit": "waypoint-queries/s", "n_gpus": world,
            "steps": len(samples), "warmup": args.warmup, "ms_per_step": 1e3 * shape.n_waypoints / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 index math + f32 lerp",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": shape.name, "waypoints": shape.n_waypoints, "points": shape.n_points},
            "cpu_baseline": {**base, "value": value},
            "e2e": {"value": value, "unit": "waypoint-queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


_T0 = time.perf_counter()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["config4", "config2", "config1"], default="config4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    dist = None
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(_env_int("LOCAL_RANK", 0))
        tdist.init_process_group("nccl")
        dist = tdist
    import paper_2309_12543_b200 as L

    out, _ = run_ours(args, rank, world, dist)
    if world == 1:
        out["realtime"] = run_realtime(args, L)
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args.workload)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
