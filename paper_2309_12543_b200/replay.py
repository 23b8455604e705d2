"""Recorded-scene replay end to end (the reference's ``run_replay``,
bench.py:410-430, with its formats query.py:313-355): a manifest of timestamped
point-cloud frames is streamed through one prepared control cycle per frame and
the per-waypoint distances are written as the reference's distance CSV.

Per frame the f32 points go straight from the frame file into the checker's
page-locked input buffer (no f64 detour on the host), the cycle runs as one
CUDA graph — the kernels read the frame zero-copy over PCIe, and (d, link,
voxel) land back in page-locked memory — and the row is kept for the CSV.
The trajectory is fixed for the whole replay, so ``materialized=True`` uses
the paper's two-phase mode instead (``MaterializedChecker``: the robot SDF of
the trajectory is assembled once, each frame is one gather).  Both give the
same distances as ``stream_min_distances`` on the same trajectory
(tests/test_gpu_benchmarked.py::test_replay_end_to_end).
"""

from __future__ import annotations

import struct
import time
from pathlib import Path

import numpy as np

from .errors import ValidationError
from .query import read_cloud_manifest, write_distance_csv

_COUNT = struct.Struct("<I")


def frame_point_count(path) -> int:
    with open(path, "rb") as fh:
        head = fh.read(_COUNT.size)
    if len(head) != _COUNT.size:
        raise ValidationError(f"{path}: truncated frame header")
    return _COUNT.unpack(head)[0]


def read_frame_into(path, out: np.ndarray) -> int:
    """Read a frame file (query.py:313-327) into ``out`` ((cap, 3) f32, NaN-padded
    past the frame's points, which the voxelizer drops); returns the count."""
    data = Path(path).read_bytes()
    (count,) = _COUNT.unpack_from(data)
    if (len(data) - _COUNT.size) // 4 < 3 * count:
        raise ValidationError(f"{path}: truncated point data")
    if count > len(out):
        raise ValidationError(f"{path}: {count} points exceed the prepared capacity {len(out)}")
    out[:count] = np.frombuffer(data, dtype="<f4", count=3 * count, offset=_COUNT.size).reshape(count, 3)
    out[count:] = np.nan
    return count


def run_replay(robot, sdfs, grid, window, configs, manifest_path, out_path, *, materialized: bool = False,
               d_far_global=None) -> dict:
    """Replay ``manifest_path`` against the trajectory ``configs`` (C, D); write
    the distance CSV to ``out_path``.  Returns the reference's summary
    (frames, min_distance_m, waypoints) plus host-to-host cycle latencies."""
    from .checker import DistanceChecker, MaterializedChecker

    entries = read_cloud_manifest(manifest_path)
    q = np.ascontiguousarray(configs, dtype=np.float64)
    cap = max([frame_point_count(p) for _, p in entries] + [1])
    if materialized:
        chk = MaterializedChecker(robot, sdfs, grid, window, q, d_far_global=d_far_global).prepare(cap, np.float32)
        pts = chk.host_points()
        cycle = chk.query
    else:
        chk = DistanceChecker(robot, sdfs, grid, window, d_far_global=d_far_global).prepare(len(q), cap, np.float32)
        q_host, pts = chk.host_inputs()
        q_host[...] = q
        cycle = chk.query
    rows, lat = [], []
    overall_min = np.inf
    for stamp, path in entries:
        read_frame_into(path, pts)  # the sensor side: file -> page-locked frame buffer (not timed)
        t0 = time.perf_counter()
        d, _, _ = cycle()
        lat.append((time.perf_counter() - t0) * 1e6)
        rows.append((stamp, d))
        if len(d):
            overall_min = min(overall_min, float(d.min()))
    write_distance_csv(out_path, rows, len(q))
    lat_a = np.asarray(lat) if lat else np.zeros(1)
    return {"frames": float(len(rows)), "min_distance_m": overall_min, "waypoints": float(len(q)),
            "cycle_p50_us": float(np.percentile(lat_a, 50)), "cycle_p99_us": float(np.percentile(lat_a, 99)),
            "mode": "materialized" if materialized else "direct"}
