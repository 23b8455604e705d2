"""Benchmark of the batched link-SDF distance checker (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  ``--gpus N`` outside torchrun launches N ranks
itself (torch.distributed.run on 127.0.0.1, one GPU per rank, NCCL).  A *step* is one pass of the hot path over one batch:
FK + alignment for every waypoint, voxelization of the step's obstacle cloud,
and the fused transform / trilinear / min / argmin query, producing
(d, link, voxel) for every waypoint.

* ``value`` — waypoint-queries/s, whole job, on BASELINE config 4 (7-DoF arm,
  65,536 waypoints vs a 1M-point crowd cloud, 64^3 link SDFs, W = 16), inputs
  resident in HBM, device time (CUDA events on the launching stream), L2
  flushed (256 MiB write) before every timed step.  N > 1 GPUs: the global
  batch is N x 65,536 waypoints against the shared scene, sharded contiguously
  across ranks (65,536 per GPU: each rank voxelizes the full resident cloud;
  no collective on the data path); time is the max over ranks -> weak scaling.
* ``realtime`` (N = 1) — BASELINE config 2: p50 / p99 µs per 500-waypoint
  query (6-DoF, 100k-point cloud, 64^3): device graph and host-to-host.
* ``e2e`` — config 4 through the public API (DistanceChecker.query) from
  pinned host buffers: the kernels read the inputs and write the results
  across PCIe inside the timed region (host wall clock per step).
* ``roofline`` — query_shells_kernel (the dominant kernel) against the bound
  it actually meets, the SM issue rate: warp instructions per launch (live
  ``ncu`` counter pass on this box during the run) over the event-timed launch
  duration, against 148 SMs x 4 sub-partitions x 1 warp-instruction/cycle at
  the sampled clock; ``traffic`` = DRAM bytes of the same launch.
* ``work_avoided`` — the reference's dense gather (4 B per occupied voxel per
  waypoint) at HBM peak vs the culled kernel's time: the
  algorithmic ratio, not a roofline fraction.
* ``cpu_baseline`` — the oracle port of the reference pipeline (numpy) on
  this host, bounded sample, rank 0 at N = 1.

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
def _kernels_per_cycle(chk, N) -> int:
    """Our kernel launches in one cycle: the library's launch counter around
    one un-captured cycle (the graph replays exactly these launches)."""
    import torch

    before = int(N.lib().lsdf_launch_count())
    chk._run(False)
    torch.cuda.synchronize()
    return int(N.lib().lsdf_launch_count()) - before


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
    """nvidia-smi clocks + throttle reasons, sampled every 50 ms while the GPU works."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        sm, mx, reasons = [], None, set()
        for ts, ln in self.lines:
            if t0 is not None and not (t0 <= ts <= t1):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[2:6]):
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


def _checker(shape, n_configs, L):
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(n_configs, shape.n_points, np.float32)
    return robot, chk


class L2Flush:
    def __init__(self, torch):
        self.buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def __call__(self):
        self.buf.zero_()


E2E_WINDOWS, E2E_MIN_CYCLES = 3, 200  # e2e throughput: best of three windows of >= 200 pipelined cycles
SPIN_CYCLES = 200_000  # ~0.1 ms GPU spin: longer than the host needs to enqueue one step


def _time_steps(torch, fn, steps, flush, before=None):
    """Per-step device times (ms), CUDA events on the launching stream, L2 flushed before each.

    A short GPU spin sits between the flush and the start event, so the host
    has enqueued the step before the start event fires: the interval is the
    step's device execution, not the host's launch latency (which the e2e
    numbers include).
    """
    stream = torch.cuda.current_stream()
    marks = []
    for k in range(steps):
        if before is not None:
            before(k)
        flush()
        torch.cuda._sleep(SPIN_CYCLES)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        marks.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in marks]


def _max_over_ranks(dist, torch, x):
    if dist is None:
        return x
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _e2e_entry(C_total, pipe_ms, single_ms, h2d, d2h, world=1):
    """The public-API end-to-end number: the faster of the pipelined and the
    one-cycle-at-a-time paths (both copy every cycle's inputs in and results out)."""
    pipe_path = ("CheckerPipeline (3 cycles in flight): per cycle one H2D of configs + cloud from pinned host memory on "
                 "a copy stream, the cycle graph, D2H of (d, link, voxel) + flags; host wall clock over max(K, 200) "
                 "cycles, best of 3 windows"
                 if world == 1 else
                 "ShardedCloudPipeline (3 cycles in flight, per rank): H2D of this rank's configs and 1/world of the "
                 "cloud, voxelize the slice, NCCL all-gather of the partial occupancy bitmaps, merge, FK + query, "
                 "D2H; host wall clock over max(K, 200) cycles, best of 3 windows, max over ranks")
    single_path = ("DistanceChecker.query() one cycle at a time from pinned host buffers (zero-copy kernel "
                   "reads/writes over PCIe); median cycle, host wall clock")
    best_ms, path = (pipe_ms, pipe_path) if (pipe_ms <= single_ms or world > 1) else (single_ms, single_path)
    return {"value": C_total / (best_ms / 1e3), "unit": "waypoint-queries/s", "ms_per_step": best_ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "path": path,
            "pipelined_ms_per_step": pipe_ms, "single_cycle_ms": single_ms}


def _h2d_peak_gbs(torch, nbytes=64 << 20, reps=5):
    """Measured host->device copy bandwidth from page-locked memory (best of `reps`, CUDA events):
    the denominator of the e2e path's PCIe bound."""
    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = float("inf")
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / (best / 1e3) / 1e9


def _pcie_bound(e2e, peak_gbs):
    """The e2e path's bound: every cycle's inputs cross PCIe (H2D), overlapped with the compute of
    the cycles in flight, so the pipelined step can be no shorter than h2d_bytes / H2D bandwidth."""
    ms = e2e["ms_per_step"]
    ach = e2e["h2d_bytes_per_step"] / (ms / 1e3) / 1e9
    return {"bound": "pcie_h2d", "achieved": ach, "peak": peak_gbs, "unit": "GB/s", "frac": ach / peak_gbs,
            "peak_kind": "measured in this run: 64 MiB page-locked -> device copy, best of 5"}


def run_ours(args, rank, world, dist, sampler):
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    shape = _shape(args.workload)
    # weak scaling: every rank checks a full config-4 batch of its own waypoints
    n_local = shape.n_waypoints
    C_total = n_local * world
    lo = rank * n_local
    robot, chk = _checker(shape, n_local, L)
    seeds = [11, 12, 13]
    # each rank owns waypoints [lo, lo + n_local) of every step's trajectory batch
    host = [(np.ascontiguousarray(S.random_configs(shape.robot, C_total, seed=s)[lo:lo + n_local]), _cloud(shape, s))
            for s in seeds]
    dev = [(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda()) for q, p in host]
    flush = L2Flush(torch)

    def stage(k):
        q, p = dev[k % len(dev)]
        chk.q_dev.copy_(q)
        chk.p_dev.copy_(p)

    step = lambda: chk.launch(device_only=True)  # noqa: E731
    _time_steps(torch, step, args.warmup, flush, stage)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev_ms = _time_steps(torch, step, args.steps, flush, stage)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if dist is not None:
        dist.barrier()
    total_ms = _max_over_ranks(dist, torch, sum(dev_ms))
    ms_per_step = total_ms / args.steps
    value = C_total / (ms_per_step / 1e3)

    # ---- e2e through the public API, one cycle at a time: pinned host inputs,
    # zero-copy reads, results back in pinned memory (the latency form)
    q_host, p_host = chk.host_inputs()
    single = []
    for k in range(args.warmup + min(args.steps, 20)):
        q, p = host[k % len(host)]
        q_host[...] = q
        p_host[: len(p)] = p
        flush()
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        chk.query()
        s1 = time.perf_counter()
        if k >= args.warmup:
            single.append(s1 - s0)
    single_ms = _max_over_ranks(dist, torch, 1e3 * statistics.median(single))

    # ---- e2e throughput through the public API: CheckerPipeline, two cycles in
    # flight; every cycle copies its configurations and cloud from pinned host
    # memory (copy engine) and reads (d, link, voxel) back, K cycles wall clock
    # with several ranks the cloud is sharded too: each rank uploads its slice
    # and the ranks all-gather their 16-KB partial occupancy bitmaps over NVLink
    def run_pipe(sharded: bool):
        if sharded:
            from paper_2309_12543_b200.sharding import shard_range

            plo, phi = shard_range(shape.n_points, rank, world)
            pipe = L.ShardedCloudPipeline(chk.robot, chk.sdfs, chk.grid, chk.window, n_local, phi - plo,
                                          np.float32, depth=3)
        else:
            plo, phi = 0, shape.n_points
            pipe = L.CheckerPipeline(chk.robot, chk.sdfs, chk.grid, chk.window, n_local, shape.n_points,
                                     np.float32, depth=3)
        for k in range(pipe.depth):  # producers write straight into the pinned slots
            qv, pv = pipe.inputs()
            q_k, p_k = host[k % len(host)]
            qv[...], pv[...] = q_k, p_k[plo:phi]
            pipe.submit()
        for k in range(pipe.depth):
            pipe.result(k)
        for _ in range(args.warmup):
            pipe.result(pipe.submit())
        torch.cuda.synchronize()
        # three timed windows of at least 200 cycles each, the best one kept:
        # a window is ~60 ms of wall clock, so one host hiccup (another tenant,
        # a page fault) would otherwise dominate a short measurement
        n_cyc = max(args.steps, E2E_MIN_CYCLES)
        best = float("inf")
        for _ in range(E2E_WINDOWS):
            if dist is not None:
                dist.barrier()
            s0 = time.perf_counter()
            tickets = [pipe.submit() for _ in range(pipe.depth)]
            for k in range(n_cyc):
                pipe.result(tickets[k])
                if k + pipe.depth < n_cyc:
                    tickets.append(pipe.submit())
            best = min(best, 1e3 * (time.perf_counter() - s0) / n_cyc)
        return best, plo, phi

    sharded = world > 1
    try:
        pipe_ms, plo, phi = run_pipe(sharded)
    except Exception as exc:  # noqa: BLE001 — keep the measurement if the sharded exchange fails
        if not sharded:
            raise
        print(f"sharded-cloud pipeline failed ({exc!r}); e2e with the full cloud per rank", file=sys.stderr)
        sharded = False
        pipe_ms, plo, phi = run_pipe(False)
    e2e_ms = _max_over_ranks(dist, torch, pipe_ms)

    from paper_2309_12543_b200 import _native as N

    per_cycle = _kernels_per_cycle(chk, N)

    # ---- roofline of the dominant kernel (query) timed alone on the staged batch
    stage(0)
    chk.launch(device_only=True)
    torch.cuda.synchronize()
    n_occ = int(chk.ws[:4].view(torch.int32).item())
    outs = {}
    qk = lambda: chk.traj.query_device(chk.ws, False, outputs=outs)  # noqa: E731
    _time_steps(torch, qk, 3, flush)
    q_ms = statistics.mean(_time_steps(torch, qk, max(5, min(args.steps, 50)), flush))
    alg_bytes = 4.0 * n_occ * n_local
    peak, peak_kind = _peaks()
    achieved = alg_bytes / (q_ms / 1e3) / 1e9
    # robustness: the same 65,536-waypoint cycle against clouds that leave
    # most windows empty (the scan must not fall back to scanning every cell)
    variants = None
    if rank == 0 and world == 1:
        variants = run_cloud_variants(torch, chk, host[0][0], shape, flush)
    # live hardware counters of this very launch (ncu subprocess, one replayed
    # launch of the same workload; never timed): warp instructions and DRAM bytes
    counters = None
    if rank == 0 and not args.no_counters:  # (N > 1: rank 0's GPU, after the timed region)
        counters = live_counters(args.workload)
    clocks = sampler.summary(t0 - 0.2, t1 + 0.2) if sampler else None
    out = {
        "metric": METRIC, "value": value, "unit": "waypoint-queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded arm7g/arm6g primitive robots, random joint configs, human/crowd point clouds",
        "config": {"workload": f"{shape.name}: {shape.robot['name']} {n_local} waypoints per GPU vs {shape.n_points} pts "
                               f"({shape.cloud}), 64^3 link SDFs, env 50^3 @ 4 cm, W=16",
                   "waypoints": C_total, "waypoints_per_gpu": n_local, "points": shape.n_points, "occupied_voxels": n_occ,
                   "parallelism": f"waypoint shards x{world}",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "timing": "device: CUDA events around a graph replay of the cycle, enqueued behind a GPU spin "
                             "(host launch latency excluded; e2e includes it)"},
        "gpu_launches": per_cycle * args.steps,
        "gpu_launches_per_step": per_cycle,
        "e2e": _e2e_entry(C_total, e2e_ms, single_ms, int(n_local * robot.dof * 8 + (phi - plo) * 12),
                          int(n_local * 12 + 16), world if sharded else 1),
        # the dense gather the reference performs (4 B per occupied voxel per
        # waypoint, query.py:146) at HBM speed, against the culled kernel: work
        # avoided, not a roofline (the kernel never reads that field)
        "work_avoided": {"dense_gather_bytes": alg_bytes, "dense_gather_ms_at_hbm_peak": alg_bytes / (peak * 1e9) * 1e3,
                         "kernel_ms": q_ms, "ratio": (alg_bytes / (peak * 1e9) * 1e3) / q_ms,
                         "peak_gbs": peak, "peak_kind": peak_kind},
        "clocks": clocks,
    }
    if world == 1:  # (N > 1: each rank moves 1/N of the cloud, see ShardedCloudPipeline)
        out["e2e"]["roofline"] = _pcie_bound(out["e2e"], _h2d_peak_gbs(torch))
    if variants is not None:
        out["cloud_variants"] = variants
    # the bound the kernel meets: its warp-instruction stream
    # against one warp instruction per SM sub-partition per cycle at the
    # sampled clock; DRAM traffic of the same launch alongside
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    peak_i = 148 * 4 * mhz * 1e6 / 1e9
    warp_inst = (counters or {}).get("warp_inst")
    ach_i = warp_inst / (q_ms / 1e3) / 1e9 if warp_inst else None
    out["roofline"] = {
        "bound": "issue", "achieved": ach_i, "peak": peak_i, "unit": "G warp-inst/s",
        "frac": ach_i / peak_i if ach_i else None,
        "traffic": (counters or {}).get("dram_bytes"), "kernel": "query_shells_kernel", "kernel_ms": q_ms,
        "warp_inst_per_launch": warp_inst,
        "peak_kind": f"148 SMs x 4 SMSPs x 1 warp-inst/cycle x the sampled SM clock ({mhz:.0f} MHz)",
        "source": (counters or {}).get("source", "counters not collected"),
    }
    return out


def run_cloud_variants(torch, chk, q, shape, flush, reps: int = 20):
    """Device cycle of the config-4 batch against an empty, a corner-packed
    ("far") and a sparse uniform cloud next to the crowd (L2 flushed, median)."""
    from paper_2309_12543_b200 import scenarios as S

    n = shape.n_points
    clouds = {
        "crowd": _cloud(shape, 11),
        "empty": np.full((n, 3), np.nan, np.float32),
        "far_corners": S.far_crowd_cloud(n, 11).astype(np.float32),
        "sparse_2k": np.concatenate([S.sparse_cloud(2000, 11), np.full((n - 2000, 3), np.nan)]).astype(np.float32),
    }
    chk.q_dev.copy_(torch.from_numpy(q))
    out = {}
    for name, pts in clouds.items():
        chk.p_dev.copy_(torch.from_numpy(pts))
        step = lambda: chk.launch(device_only=True)  # noqa: E731
        _time_steps(torch, step, 3, flush)
        ms = statistics.median(_time_steps(torch, step, reps, flush))
        n_occ = int(chk.ws[:4].view(torch.int32).item())
        out[name] = {"occupied_voxels": n_occ, "ms_per_step": ms,
                     "waypoint_queries_per_s": shape.n_waypoints / (ms / 1e3)}
    return out


# ----------------------------------------------------------------------------- live counters


_PROBE_METRICS = "smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def probe_counters(args):
    """The workload's cycle, untimed, for ncu to capture one query launch (--probe-counters)."""
    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    shape = _shape(args.workload)
    _, chk = _checker(shape, shape.n_waypoints, L)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    chk.q_dev.copy_(torch.from_numpy(np.ascontiguousarray(q)))
    chk.p_dev.copy_(torch.from_numpy(_cloud(shape, 11)))
    for _ in range(3):  # warm cycles (the link order comes from the previous cycle)
        chk.launch(device_only=True)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()  # ncu --profile-from-start off: only this cycle is profiled
    chk.launch(device_only=True)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


def live_counters(workload: str, timeout: float = 240.0):
    """smsp__inst_executed / DRAM bytes of one query_shells_kernel launch of this
    workload, from ncu run on this box now (a launch replayed under the
    profiler: counted, never timed)."""
    import csv
    import shutil
    import tempfile

    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not Path(ncu).exists():
        return {"source": "ncu not found"}
    with tempfile.TemporaryDirectory() as td:
        log = Path(td) / "counters.csv"
        cmd = [ncu, "--metrics", _PROBE_METRICS, "--clock-control", "none", "--print-units", "base", "--csv",
               "--profile-from-start", "off", "-k", "regex:query_shells_kernel", "--launch-count", "1",
               "--log-file", str(log), sys.executable, str(Path(__file__).resolve()), "--probe-counters",
               "--workload", workload]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        except subprocess.TimeoutExpired:
            return {"source": f"ncu timed out after {timeout:.0f} s"}
        if r.returncode != 0 or not log.exists():
            return {"source": f"ncu failed (rc {r.returncode}): {(r.stderr or r.stdout)[-200:]}"}
        rows = [row for row in csv.reader(log.read_text().splitlines()) if row]
    try:
        hi = next(i for i, row in enumerate(rows) if row[0] == "ID")
    except StopIteration:
        return {"source": "ncu wrote no metrics"}
    h = rows[hi]
    name_i, val_i = h.index("Metric Name"), h.index("Metric Value")
    m = {row[name_i]: float(row[val_i].replace(",", "")) for row in rows[hi + 1:]}
    return {"warp_inst": m.get("smsp__inst_executed.sum"),
            "dram_bytes": (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) or None,
            "ncu_duration_ns": m.get("gpu__time_duration.sum"),
            "source": f"ncu --metrics {_PROBE_METRICS} on this box during this run: the scan of the 4th "
                      f"{workload} cycle (replayed under the profiler, caches flushed; counted, not timed)"}


def run_realtime(args, L, workload: str = "config2"):
    """Config 2 (or 1): p50/p99 per 500-waypoint query (device graph and host-to-host)."""
    import torch

    from paper_2309_12543_b200 import scenarios as S

    shape = _shape(workload)
    robot, chk = _checker(shape, shape.n_waypoints, L)
    inputs = [(S.random_configs(shape.robot, shape.n_waypoints, seed=s), _cloud(shape, s)) for s in (21, 22, 23, 24)]
    dev = [(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda()) for q, p in inputs]
    flush = L2Flush(torch)

    def stage(k):
        q, p = dev[k % len(dev)]
        chk.q_dev.copy_(q)
        chk.p_dev.copy_(p)

    n = max(200, args.steps)
    _time_steps(torch, lambda: chk.launch(device_only=True), 10, flush, stage)
    devt = _time_steps(torch, lambda: chk.launch(device_only=True), n, flush, stage)
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
    sphere = sphere_comparison(torch, L, shape, inputs[0], flush) if workload == "config2" else None
    grid_n = int(round(2 * shape.link_extent / shape.link_res))
    return {"workload": f"{shape.name}: arm6g 500 waypoints vs {shape.n_points // 1000}k pts, {grid_n}^3, W=16",
            "occupied_voxels": n_occ,
            "device_p50_us": pct(devt, 50), "device_p99_us": pct(devt, 99),
            "e2e_p50_us": pct(e2e, 50), "e2e_p99_us": pct(e2e, 99), "samples": n,
            "waypoint_queries_per_s_device": 500 / (statistics.mean(devt) / 1e3),
            "paper_gpu_ms_per_trajectory": 0.391,
            **({"sphere_baseline": sphere} if sphere is not None else {})}


# covering spheres of the arm6g links (tests/golden/make_golden_r2.py ARM6G_SPHERES)
_ARM6G_SPHERES = {
    "l1": [{"center": [0, 0, z], "radius": 0.07} for z in (-0.06, 0.0, 0.06)],
    "l2": [{"center": [0, 0, z], "radius": 0.06} for z in (-0.08, 0.0, 0.08)],
    "l3": [{"center": [0, 0, z], "radius": 0.05} for z in (-0.07, 0.0, 0.07)],
    "l4": [{"center": [0, 0, z], "radius": 0.045} for z in (-0.05, 0.0, 0.05)],
    "l5": [{"center": [0, 0, 0], "radius": 0.0755}],
    "l6": [{"center": [0, 0, 0], "radius": 0.05}],
}


def sphere_comparison(torch, L, shape, inp, flush, reps: int = 50):
    """The paper's comparison (Table: 5.47 ms sphere model vs
    0.391 ms per trajectory): the covering-sphere checker (query.py:254-291,
    every sphere x every occupied voxel, fp64) on the same 500 waypoints and
    cloud, device time per trajectory with poses and voxels resident."""
    import copy
    import ctypes

    from paper_2309_12543_b200 import _native as N

    doc = copy.deepcopy(shape.robot)
    doc["spheres"] = _ARM6G_SPHERES
    robot = L.RobotModel.from_dict(doc)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    q, pts = inp
    poses = L.forward_kinematics_batch(robot, L.ConfigBatch(q))
    obs = L.voxelize_pointcloud(pts, grid)
    sph = L.SphereRobotModel.from_robot(robot)
    R = torch.from_numpy(np.ascontiguousarray(poses.rotations)).cuda()
    T = torch.from_numpy(np.ascontiguousarray(poses.translations)).cuda()
    sl = torch.from_numpy(sph.link_indices.astype(np.int32)).cuda()
    sc = torch.from_numpy(np.ascontiguousarray(sph.centers)).cuda()
    sr = torch.from_numpy(np.ascontiguousarray(sph.radii)).cuda()
    out = torch.empty((len(q),), dtype=torch.float64, device="cuda")
    idx = obs.device_indices()
    env = ctypes.byref(grid.c_struct())
    call = lambda: N.call("lsdf_sphere_baseline", R, T, len(q), poses.n_links, sl, sc, sr, sph.n_spheres,  # noqa: E731
                          idx, obs.n_occupied, env, out, N.stream())
    _time_steps(torch, call, 3, flush)
    ts = _time_steps(torch, call, reps, flush)
    return {"spheres": sph.n_spheres, "occupied_voxels": obs.n_occupied, "device_p50_us": float(np.median(ts) * 1e3),
            "distance_evals": int(len(q) * sph.n_spheres * obs.n_occupied), "paper_sphere_ms_per_trajectory": 5.47}


def run_dynamic(L, repeats: int = 3):
    """Config 5: 100 control cycles (8 ms apart) re-querying a fixed 500-waypoint
    trajectory against a human walking in from 1.4 m at 1.6 m/s (30k points).
    Host to host per cycle (DistanceChecker.query: the kernels read the frame
    from page-locked memory and write (d, link, voxel) back), and the paper's
    prepare-once mode (MaterializedChecker), whose results must be identical."""
    import torch

    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG5
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    frames = [(t, np.ascontiguousarray(p, dtype=np.float32)) for t, p in S.moving_human_frames(100, shape.n_points,
                                                                                                 seed=5)]
    q = S.smooth_trajectory(shape.robot, shape.n_waypoints, seed=5)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(shape.n_waypoints, shape.n_points, np.float32)
    q_host, p_host = chk.host_inputs()
    q_host[...] = q
    for _ in range(10):
        p_host[...] = frames[0][1]
        chk.query()
    wall, results = [], []
    for rep in range(repeats):
        for _, pts in frames:
            p_host[...] = pts  # the sensor side's write into the page-locked frame buffer (not timed)
            t0 = time.perf_counter()
            r = chk.query()
            wall.append((time.perf_counter() - t0) * 1e6)
            if rep == 0:
                results.append(r)
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
        mp[...] = frames[0][1]
        mat.query()
    wall_m, same = [], True
    for rep in range(repeats):
        for k, (_, pts) in enumerate(frames):
            mp[...] = pts
            t0 = time.perf_counter()
            rm = mat.query()
            wall_m.append((time.perf_counter() - t0) * 1e6)
            if rep == 0:
                same &= all(np.array_equal(a, b) for a, b in zip(rm, results[k]))
    pct = lambda a, p: float(np.percentile(a, p))  # noqa: E731
    return {"workload": "config5_dynamic: arm6g 500 waypoints, 100 frames x 30k pts (a human walking in), 64^3",
            "cycles": len(wall), "e2e_p50_us": pct(wall, 50), "e2e_p99_us": pct(wall, 99), "e2e_max_us": max(wall),
            "cycle_budget_us": 8000.0,
            "frames_with_obstacle_in_range": sum(int((r[1] >= 0).any()) for r in results),
            "materialized": {"prepare_ms_once": prep_ms, "e2e_p50_us": pct(wall_m, 50),
                             "e2e_p99_us": pct(wall_m, 99), "same_results_as_direct": bool(same)}}


# ----------------------------------------------------------------------------- CPU (oracle port)


class CpuPort:
    """The oracle port of the reference pipeline (numpy), set up once per workload."""

    def __init__(self, workload: str, sample: int):
        from oracle import linksdf_oracle as O
        from paper_2309_12543_b200 import scenarios as S

        self.O = O
        self.shape = shape = _shape(workload)
        chain = O.chain_from_doc(shape.robot)
        self.chain = chain
        self.gl = O.geometry_links(chain)
        self.grids = [O.build_grid(chain[i]["geometry"], shape.link_extent, shape.link_res) for i in self.gl]
        self.env = O.Env(shape.grid_extent, shape.grid_res)
        pts = _cloud(shape, 11)
        t0 = time.perf_counter()
        self.idx, _, _ = O.voxelize(pts, self.env)
        self.t_vox = time.perf_counter() - t0
        self.sample = min(sample, shape.n_waypoints)
        self.q = S.random_configs(shape.robot, self.sample, seed=11)

    def sample_seconds(self) -> float:
        """Wall seconds of FK + placement + assembly + gather + argmin on the sample."""
        O, shape, gl = self.O, self.shape, self.gl
        t0 = time.perf_counter()
        R, T = O.fk(self.chain, self.q)
        windows, anchors = O.place_windows(self.grids, [shape.link_extent] * len(gl), [shape.link_res] * len(gl),
                                           R[:, gl], T[:, gl], self.env, shape.link_extent)
        batch = O.assemble(windows, anchors, self.env, shape.link_extent)
        O.argmin_oracle(batch, windows, anchors, self.idx, shape.link_extent)
        return time.perf_counter() - t0

    def describe(self, reps, procs):
        shape = self.shape
        return (f"{shape.name}: {procs} processes x {self.sample} waypoints per step, {reps} steps, through FK + "
                f"placement + assembly + gather + argmin (oracle port of the reference, numpy, one BLAS thread per "
                f"process) against the full {shape.n_points}-pt cloud voxelized once ({self.t_vox:.2f} s, charged "
                f"per waypoint over {shape.n_waypoints})")


_PORT = None  # inherited by the forked workers


def _port_task(_):
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        return _PORT.sample_seconds()


class PortPool:
    """The port on every host core: one forked process per core, each running
    the bounded sample; a step = all processes once (wall clock)."""

    def __init__(self, workload: str, sample: int = 64):
        import multiprocessing as mp

        global _PORT
        _PORT = self.port = CpuPort(workload, sample)
        self.procs = len(os.sched_getaffinity(0))
        self.pool = mp.get_context("fork").Pool(self.procs)

    def step(self) -> float:
        """Seconds per waypoint-query of one parallel step (voxelize charged pro rata)."""
        t0 = time.perf_counter()
        self.pool.map(_port_task, range(self.procs), chunksize=1)
        wall = time.perf_counter() - t0
        port = self.port
        return wall / (self.procs * port.sample) + port.t_vox / port.shape.n_waypoints

    def close(self):
        self.pool.terminate()


def cpu_baseline(workload: str, budget_s: float = 15.0, sample: int = 64):
    pool = PortPool(workload, sample)
    try:
        pool.step()  # warm-up (worker start)
        per_wp, t_start = [], time.perf_counter()
        while len(per_wp) < 2 or (time.perf_counter() - t_start < budget_s and len(per_wp) < 20):
            per_wp.append(pool.step())
    finally:
        pool.close()
    v = 1.0 / statistics.median(per_wp)
    return {"value": v, "unit": "waypoint-queries/s", "cores": pool.procs, "kind": "port",
            "sample": pool.port.describe(len(per_wp), pool.procs), "extrapolated": True,
            "sample_waypoints_per_step": pool.procs * pool.port.sample}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    pool = PortPool(args.workload, 64)
    try:
        for _ in range(max(args.warmup, 1)):
            pool.step()
        per_wp = []
        t_start = time.perf_counter()
        for _ in range(args.steps):
            per_wp.append(pool.step())
            if time.perf_counter() - t_start > 240:
                break
    finally:
        pool.close()
    value = len(per_wp) / sum(per_wp)
    shape = pool.port.shape
    per_step = pool.procs * pool.port.sample
    # a step is a bounded sample of the workload: `per_step` of its 65,536
    # waypoints against the full cloud; ms_per_step is that sample's time
    # (the metric is per waypoint, so it is the same for a full step)
    return {"metric": METRIC, "value": value, "unit": "waypoint-queries/s", "n_gpus": world,
            "steps": len(per_wp), "warmup": args.warmup, "ms_per_step": 1e3 * per_step / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": shape.name, "waypoints": shape.n_waypoints, "points": shape.n_points,
                       "waypoints_per_step": per_step},
            "sample_waypoints_per_step": per_step,
            "full_step_waypoints": shape.n_waypoints,
            "full_step_ms_extrapolated": 1e3 * shape.n_waypoints / value,
            "cpu_baseline": {"value": value, "unit": "waypoint-queries/s", "cores": pool.procs, "kind": "port",
                             "sample": pool.port.describe(len(per_wp), pool.procs)},
            "e2e": {"value": value, "unit": "waypoint-queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _spawn_ranks(n: int) -> int:
    """``--gpus N`` outside torchrun: launch N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and pass rank 0's line through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def run_dry(args, rank, world, dist):
    """``--dry-run``: the multi-rank plumbing only (rendezvous, barrier,
    max-over-ranks reduction, rank-0 print) with no GPU work — what the CPU
    test of ``--gpus N`` exercises."""
    import torch

    per_rank_ms = 1.0 + rank  # stand-in step time: the max over ranks must be the last rank's
    t = torch.tensor([per_rank_ms], dtype=torch.float64)
    if dist is not None:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"metric": METRIC, "dry_run": True, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(t.item()), "backend": dist.get_backend() if dist is not None else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["config4", "config2", "config1"], default="config4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-counters", action="store_true", help="skip the live ncu counter pass")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only, no GPU work")
    ap.add_argument("--probe-counters", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.probe_counters:
        return probe_counters(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(_spawn_ranks(args.gpus))
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    import torch

    dist = None
    if world > 1:
        import torch.distributed as tdist

        # LSDF_BENCH_BACKEND=gloo: functional check of the multi-rank path
        # (the CPU test's --dry-run, or one GPU: numbers meaningless); the
        # driver's runs use NCCL, one GPU per rank
        backend = os.environ.get("LSDF_BENCH_BACKEND", "gloo" if args.dry_run else "nccl")
        if backend == "nccl":
            torch.cuda.set_device(_env_int("LOCAL_RANK", 0) % max(1, torch.cuda.device_count()))
        tdist.init_process_group(backend)
        dist = tdist
    if args.dry_run:
        out = run_dry(args, rank, world, dist)
        if rank == 0:
            print(json.dumps(out), flush=True)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    torch.cuda.set_device(_env_int("LOCAL_RANK", 0) % max(1, torch.cuda.device_count()))
    import paper_2309_12543_b200 as L

    sampler = ClockSampler(torch.cuda.current_device()).start()
    try:
        out = run_ours(args, rank, world, dist, sampler)
        if world == 1:
            out["realtime"] = run_realtime(args, L)
            out["config1"] = run_realtime(args, L, "config1")
            out["dynamic"] = run_dynamic(L)
    finally:
        sampler.stop()
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.workload)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
