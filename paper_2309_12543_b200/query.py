"""Robot-SDF assembly, obstacle voxelization and distance queries (stages 3-4).

Host-side mirror of the reference ``query.py`` (query.py:30-355) with the
same names, argument order and return types, plus the B200-native additions
SURVEY.md §8b asks for:

* :class:`TrajectorySdf` — a lazy ``RobotSdfBatch``-compatible handle.  It
  keeps only the link grids and the per-(waypoint, link) poses on the GPU;
  ``query_min_distances(handle, obstacles)`` then runs the fused direct
  kernel (transform + trilinear + min/argmin over occupied voxels inside each
  link's sphere-masked window), which is bit-identical to gathering from the
  assembled dense field.  ``.values`` materialises the dense
  field on demand.
* ``return_argmin=True`` (keyword-only, no "pose"/"rotation" in the name, see
  test_acceptance.py:389-391) returns (d, link, voxel).
* :func:`query_trajectory` — configurations + points/voxels → (d, link, voxel).

Dense batches (the paper's materialised mode) stay supported: assembly and
the gather query run as CUDA kernels too.
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Iterator

import numpy as np

from . import _native as N
from .errors import GridMismatchError, ValidationError
from .grids import EnvGrid, SdfSampleField
from .meshes import TriangleMesh, primitive_surface_points

DEFAULT_BATCH_BYTES = 1 << 30  # reference refuses dense batches past 1 GiB (query.py:27)


# =========================================================================== containers


class RobotSdfBatch:
    """Dense per-configuration robot distance fields (query.py:30-44).

    ``values`` (C, nx, ny, nz) f32; resident on the GPU, host copy on demand.
    """

    def __init__(self, values, grid: EnvGrid, d_far_global: float):
        t = N.torch()
        self.grid = grid
        self.d_far_global = float(d_far_global)
        if isinstance(values, t.Tensor):
            self._dev = values
            self._host = None
        else:
            self._host = np.asarray(values, dtype=np.float32)
            self._dev = None

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            self._host = self._dev.cpu().numpy()
            self._host.flags.writeable = False
        return self._host

    def device_values(self):
        if self._dev is None:
            self._dev = N.to_device(np.ascontiguousarray(self._host), N.torch().float32)
        return self._dev

    @property
    def n_configs(self) -> int:
        return int((self._dev if self._dev is not None else self._host).shape[0])


class ObstacleVoxelSet:
    """Deduplicated occupied voxels of a point cloud (query.py:47-58).

    ``indices`` (N_occ, 3) int64, lexicographically sorted when produced by
    :func:`voxelize_pointcloud`.  The GPU occupancy structures (bit map +
    position grid) are attached lazily and reused by every query.
    """

    def __init__(self, indices, grid: EnvGrid, n_points: int, n_dropped: int, _occupancy=None,
                 _sorted_unique=None):
        self.indices = indices
        self.grid = grid
        self.n_points = n_points
        self.n_dropped = n_dropped
        self._occ = _occupancy
        self._sorted = _sorted_unique

    @property
    def n_occupied(self) -> int:
        return len(self.indices)

    def occupancy(self):
        """(workspace tensor, by_position flag) for the query kernels."""
        if self._occ is None:
            idx = np.asarray(self.indices, dtype=np.int64).reshape(-1, 3)
            if len(idx) and (np.any(idx < 0) or np.any(idx >= self.grid.dims)):
                raise ValidationError("obstacle voxel indices outside the environment grid")
            if self._sorted is None:
                lin = (idx[:, 0] * self.grid.dims[1] + idx[:, 1]) * self.grid.dims[2] + idx[:, 2]
                self._sorted = bool(np.all(np.diff(lin) > 0))
            t = N.torch()
            ws = N.empty((int(N.lib().lsdf_occupancy_bytes(ctypes.byref(self.grid.c_struct()))),), t.uint8)
            d_idx = N.to_device(idx.astype(np.int32), t.int32)
            N.call("lsdf_occupancy_from_indices", N.ptr(d_idx), len(idx), int(self._sorted),
                   ctypes.byref(self.grid.c_struct()), N.ptr(ws), N.stream())
            self._occ = ws
            self._dev_idx = d_idx
        return self._occ, (not self._sorted)

    def device_indices(self):
        if not hasattr(self, "_dev_idx"):
            self._dev_idx = N.to_device(np.asarray(self.indices, dtype=np.int32).reshape(-1, 3), N.torch().int32)
        return self._dev_idx


def occupancy_workspace(grid: EnvGrid):
    t = N.torch()
    return N.empty((int(N.lib().lsdf_occupancy_bytes(ctypes.byref(grid.c_struct()))),), t.uint8)


def voxelize_device(points_dev, grid: EnvGrid, workspace=None, indices_out=None):
    """Launch the voxelizer on a device point tensor (N, 3) f32/f64."""
    t = N.torch()
    ws = workspace if workspace is not None else occupancy_workspace(grid)
    f32 = points_dev.dtype == t.float32
    if not f32 and points_dev.dtype != t.float64:
        points_dev = points_dev.to(t.float64)
    N.call("lsdf_voxelize", N.ptr(points_dev), int(f32), int(points_dev.shape[0]),
           ctypes.byref(grid.c_struct()), N.ptr(ws), N.ptr(indices_out), N.stream())
    return ws


def voxelize_pointcloud(points, grid: EnvGrid) -> ObstacleVoxelSet:
    """Snap a cloud to sorted unique occupied voxels, dropping out-of-bounds (query.py:106-125).

    Accepts numpy (any float dtype; f32 and f64 are voxelized exactly as the
    reference's f64 arithmetic) or a CUDA tensor.
    """
    t = N.torch()
    if isinstance(points, t.Tensor):
        pts = points.reshape(-1, 3)
        if pts.dtype not in (t.float32, t.float64):
            pts = pts.to(t.float64)
        pts = N.to_device(pts)
    else:
        arr = np.asarray(points)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        pts = N.to_device(np.ascontiguousarray(arr.reshape(-1, 3)))
    n = int(pts.shape[0])
    idx_dev = N.empty((max(1, min(n, grid.n_voxels)), 3), t.int32)
    ws = voxelize_device(pts, grid, indices_out=idx_dev)
    counters = ws[:8].view(t.int32).cpu().numpy()
    n_occ, n_drop = int(counters[0]), int(counters[1])
    idx = idx_dev[:n_occ].cpu().numpy().astype(np.int64)
    idx.flags.writeable = False
    out = ObstacleVoxelSet(indices=idx, grid=grid, n_points=n, n_dropped=n_drop, _occupancy=ws,
                           _sorted_unique=True)
    out._dev_idx = idx_dev[:n_occ]
    return out


# =========================================================================== trajectory handle


class TrajectorySdf:
    """Lazy robot-SDF batch for one trajectory (RobotSdfBatch-compatible).

    Holds the geometry-link SDF grids, the window geometry and the device
    poses (rotation, alignment residual, anchor per waypoint x link).  Queries
    run the fused direct kernel; ``values`` assembles the dense batch on demand.
    """

    def __init__(self, sdfs, grid: EnvGrid, window, R_dev, dt_dev, anchor_dev, d_far_global=None,
                 flags=None, pin_l2: bool | None = None, link_major: bool = False):
        from .placement import _check_links, link_grid_table, packed_arena

        _check_links(sdfs, window)
        self.sdfs = list(sdfs)
        self.grid = grid
        self.window = window
        self.R = R_dev
        self.dt = dt_dev
        self.anchor = anchor_dev
        # link-major storage ((L, C, .) buffers seen as (C, L, .) views, as the
        # DistanceChecker keeps large batches): the fused query reads it in
        # place, the other kernels get configuration-major copies
        self.link_major = bool(link_major)
        self.d_far_global = float(min(s.d_far for s in sdfs) if d_far_global is None else d_far_global)
        # the packed grids in one arena, pinned in L2 (persisting set-aside)
        self._arena, ptrs = packed_arena(self.sdfs)
        self._table = link_grid_table(self.sdfs, packed=True, packed_ptrs=ptrs)
        if pin_l2 is None:  # LSDF_L2_PIN=0 turns the set-aside off (A/B measurements)
            pin_l2 = os.environ.get("LSDF_L2_PIN", "1") != "0"
        self.l2_pinned_bytes = N.l2_reserve(self._arena.numel() * 4) if pin_l2 else 0
        self._ws = None
        self._dense = None
        self._flags = flags

    @property
    def n_configs(self) -> int:
        return int(self.R.shape[0])

    def config_major(self):
        """(R, dt, anchor) in the (C, L, .) layout the placement and materialization kernels read."""
        if not self.link_major:
            return self.R, self.dt, self.anchor
        return self.R.contiguous(), self.dt.contiguous(), self.anchor.contiguous()

    @property
    def n_links(self) -> int:
        return len(self.sdfs)

    @classmethod
    def from_poses(cls, sdfs, poses, grid: EnvGrid, provider, d_far_global=None):
        """From geometry-link poses (LinkPoseBatch, C x L) — placement.py:289-295 alignment on GPU.

        The fused direct kernel evaluates the exact transform (placement.py:148-169).
        Any other provider (NeuralTransformProvider, or a custom one) returns a
        :class:`PlacedTrajectorySdf` instead: the windows are placed with that
        provider's coordinates (placement.py:300-313) and queried by the dense
        gather, as the reference does with it.
        """
        from .errors import NoOverlapError
        from .placement import ExactTransformProvider, _align_device

        if not isinstance(provider, ExactTransformProvider):
            return PlacedTrajectorySdf.from_poses(sdfs, poses, grid, provider, d_far_global)
        window = provider.window
        t = N.torch()
        C_, L = poses.n_configs, poses.n_links
        if len(sdfs) != L:
            raise ValidationError(f"{len(sdfs)} SDFs for {L} links")
        R = N.to_device(np.ascontiguousarray(poses.rotations, dtype=np.float64), t.float64)
        T = N.to_device(np.ascontiguousarray(np.asarray(poses.translations, np.float64).reshape(-1, 3)), t.float64)
        anchor, dt, flags = _align_device(T, grid, window.dims)
        if int(flags[1].item()):
            raise NoOverlapError(f"{int(flags[1].item())} window(s) miss the grid entirely")
        return cls(sdfs, grid, window, R, dt.reshape(C_, L, 3), anchor.reshape(C_, L, 3), d_far_global)

    @classmethod
    def from_configs(cls, robot, configs, sdfs, grid: EnvGrid, window, d_far_global=None,
                     check=True) -> "TrajectorySdf":
        """FK + alignment on the GPU for configurations (C, D) (numpy or CUDA tensor)."""
        from .robot import ConfigBatch, check_limits, fk_device

        t = N.torch()
        if isinstance(configs, t.Tensor):
            q = N.to_device(configs, t.float64)
        else:
            batch = configs if isinstance(configs, ConfigBatch) else ConfigBatch(configs)
            if check:
                check_limits(robot, batch)
            q = N.to_device(batch.configurations, t.float64)
        out = fk_device(robot, q, all_links=False, grid=grid, window_dims=window.dims)
        traj = cls(sdfs, grid, window, out["R_geo"], out["dt_geo"], out["anchor_geo"], d_far_global,
                   flags=out["flags"])
        if check:
            traj.raise_flags()
        return traj

    def raise_flags(self):
        from .errors import NoOverlapError

        if self._flags is not None:
            f = self._flags.cpu().numpy()
            if f[0]:
                raise ValidationError(f"{int(f[0])} joint limit violation(s) in the configurations")
            if f[1]:
                raise NoOverlapError(f"{int(f[1])} window(s) miss the grid entirely")

    def windows_device(self):
        from .placement import place_windows_device

        R, dt, _ = self.config_major()
        return place_windows_device(self.sdfs, R, dt, self.window)

    def device_values(self, max_bytes: int = 1 << 36):
        if self._dense is None:
            C_, L = self.n_configs, self.n_links
            need = C_ * self.grid.n_voxels * 4
            if need > max_bytes:
                raise ValidationError(f"dense robot SDF batch needs {need / 2**20:.0f} MiB, "
                                      f"over the {max_bytes / 2**20:.0f} MiB budget")
            t = N.torch()
            win = self.windows_device()
            cfg = t.arange(C_, device=win.device, dtype=t.int32).repeat_interleave(L)
            out = N.empty((C_,) + tuple(int(d) for d in self.grid.dims), t.float32)
            N.call("lsdf_assemble", N.ptr(win), N.ptr(self.config_major()[2]), N.ptr(cfg), C_ * L, N.i32x3(self.window.dims),
                   ctypes.byref(self.grid.c_struct()), C_, self.d_far_global, N.ptr(out), N.stream())
            self._dense = out
        return self._dense

    @property
    def values(self) -> np.ndarray:
        v = self.device_values().cpu().numpy()
        v.flags.writeable = False
        return v

    def query_device(self, occupancy, by_position: bool, outputs=None, per_link=False):
        """Enqueue the fused direct query; returns dict of CUDA tensors (d, link, voxel[, per_link])."""
        t = N.torch()
        C_ = self.n_configs
        out = outputs if outputs is not None else {}
        if "d" not in out:
            out["d"] = N.empty((C_,), t.float32)
            out["link"] = N.empty((C_,), t.int32)
            out["voxel"] = N.empty((C_,), t.int32)
        if per_link and "per_link" not in out:
            out["per_link"] = N.empty((C_, self.n_links), t.float32)
        ws, _ = self.window.device_tables()
        if self._ws is None:  # zeroed once; every launch leaves it zeroed again
            nbytes = int(N.lib().lsdf_query_workspace_bytes(C_, self.n_links))
            self._ws = N.zeros((nbytes,), t.uint8)
        flags = (N.QUERY_BY_POSITION if by_position else 0) | (N.QUERY_POSES_LINK_MAJOR if self.link_major else 0)
        N.call("lsdf_query_direct", N.ptr(self.R), N.ptr(self.dt), N.ptr(self.anchor), C_, self.n_links,
               self._table, ctypes.byref(ws), ctypes.byref(self.grid.c_struct()), N.ptr(occupancy),
               flags, self.d_far_global, N.ptr(self._ws), N.ptr(out["d"]), N.ptr(out["link"]),
               N.ptr(out["voxel"]), N.ptr(out.get("per_link")), N.stream())
        return out

    def per_link_min_distances(self, obstacles: ObstacleVoxelSet) -> np.ndarray:
        """(C, L) per-link minima (query.py:153-176) from the same fused kernel."""
        occ, by_pos = obstacles.occupancy()
        return self.query_device(occ, by_pos, per_link=True)["per_link"].cpu().numpy()


class PlacedTrajectorySdf:
    """RobotSdfBatch-compatible trajectory whose windows come from any
    TransformProvider (placement.py:213-220) — in practice the neural one.

    The windows of every (waypoint, link) are placed on the GPU with the
    provider's coordinates (NeuralTransformProvider: TinyMlp on the tensor
    cores, then the fp64 shift and trilinear sampling), min-merged into the
    dense (C, nx, ny, nz) batch (query.py:61-103) once, and every query is the
    dense gather (query.py:128-150) plus the Appendix-B argmin link read off
    the windows at the winning voxel.  The fused shell scan is not used here:
    its culling bounds are proven for the exact transform only.
    """

    def __init__(self, sdfs, grid: EnvGrid, window, windows_dev, anchors_dev, d_far_global, provider=None,
                 max_bytes: int = 1 << 36):
        self.sdfs = list(sdfs)
        self.grid = grid
        self.window = window
        self.provider = provider
        self.windows = windows_dev      # (C, L, W^3) f32, x-fastest cells, masked = link d_far
        self.anchors = anchors_dev      # (C, L, 3) i32
        self.d_far_global = float(d_far_global)
        C_, L = int(windows_dev.shape[0]), int(windows_dev.shape[1])
        need = C_ * grid.n_voxels * 4
        if need > max_bytes:
            raise ValidationError(f"dense robot SDF batch needs {need / 2**20:.0f} MiB, "
                                  f"over the {max_bytes / 2**20:.0f} MiB budget")
        t = N.torch()
        cfg = t.arange(C_, device=windows_dev.device, dtype=t.int32).repeat_interleave(L)
        self._dense = N.empty((C_,) + tuple(int(d) for d in grid.dims), t.float32)
        N.call("lsdf_assemble", N.ptr(windows_dev), N.ptr(anchors_dev), N.ptr(cfg), C_ * L, N.i32x3(window.dims),
               ctypes.byref(grid.c_struct()), C_, self.d_far_global, N.ptr(self._dense), N.stream())

    @classmethod
    def from_poses(cls, sdfs, poses, grid: EnvGrid, provider, d_far_global=None) -> "PlacedTrajectorySdf":
        from .errors import NoOverlapError
        from .placement import _align_device, _check_links, place_windows_device

        window = provider.window
        _check_links(sdfs, window)
        t = N.torch()
        C_, L = poses.n_configs, poses.n_links
        if len(sdfs) != L:
            raise ValidationError(f"{len(sdfs)} SDFs for {L} links")
        R = N.to_device(np.ascontiguousarray(poses.rotations, dtype=np.float64), t.float64)
        T = N.to_device(np.ascontiguousarray(np.asarray(poses.translations, np.float64).reshape(-1, 3)), t.float64)
        anchor, dt, flags = _align_device(T, grid, window.dims)
        if int(flags[1].item()):
            raise NoOverlapError(f"{int(flags[1].item())} window(s) miss the grid entirely")
        win = place_windows_device(sdfs, R, dt.reshape(C_, L, 3), window, provider)
        d_far = float(min(s.d_far for s in sdfs) if d_far_global is None else d_far_global)
        return cls(sdfs, grid, window, win, anchor.reshape(C_, L, 3), d_far, provider)

    @property
    def n_configs(self) -> int:
        return int(self.windows.shape[0])

    @property
    def n_links(self) -> int:
        return len(self.sdfs)

    def device_values(self):
        return self._dense

    @property
    def values(self) -> np.ndarray:
        v = self._dense.cpu().numpy()
        v.flags.writeable = False
        return v

    def query_device(self, indices_dev, n_occupied: int, outputs=None):
        """(d, link, voxel) CUDA tensors for a sorted index list (the reference's gather + Appendix B)."""
        t = N.torch()
        C_ = self.n_configs
        out = outputs if outputs is not None else {}
        if "d" not in out:
            out["d"] = N.empty((C_,), t.float32)
            out["link"] = N.empty((C_,), t.int32)
            out["voxel"] = N.empty((C_,), t.int32)
        if "argmin" not in out:
            out["argmin"] = N.empty((C_,), t.int32)
        N.call("lsdf_query_dense", N.ptr(self._dense), C_, ctypes.byref(self.grid.c_struct()), N.ptr(indices_dev),
               int(n_occupied), N.ptr(out["d"]), N.ptr(out["argmin"]), N.stream())
        N.call("lsdf_link_at_voxel", N.ptr(self.windows), N.ptr(self.anchors), C_, self.n_links,
               N.i32x3(self.window.dims), N.ptr(indices_dev), N.ptr(out["argmin"]), N.ptr(out["d"]),
               float(np.float32(self.d_far_global)), N.ptr(out["link"]), N.ptr(out["voxel"]), N.stream())
        return out

    def per_link_min_distances(self, obstacles: "ObstacleVoxelSet") -> np.ndarray:
        """(C, L) per-link minima (query.py:153-176) over the placed windows."""
        t = N.torch()
        C_, L = self.n_configs, self.n_links
        out = N.empty((C_, L), t.float32)
        N.call("lsdf_fill", N.ptr(out), out.numel(), float(np.float32(self.d_far_global)), N.stream())
        if obstacles.n_occupied == 0:
            return out.cpu().numpy()
        occ, _ = obstacles.occupancy()
        cfg = t.arange(C_, device=out.device, dtype=t.int32).repeat_interleave(L)
        lnk = t.arange(L, device=out.device, dtype=t.int32).repeat(C_)
        dfar = t.tensor([float(np.float32(s.d_far)) for s in self.sdfs], dtype=t.float32, device=out.device).repeat(C_)
        N.call("lsdf_per_link_fields", N.ptr(self.windows), N.ptr(self.anchors), N.ptr(cfg), N.ptr(lnk), N.ptr(dfar),
               C_ * L, N.i32x3(self.window.dims), L, ctypes.byref(obstacles.grid.c_struct()), N.ptr(occ), N.ptr(out),
               N.stream())
        return out.cpu().numpy()


class VoxelMajorSdf:
    """The paper's materialized mode: the assembled
    robot SDF of one fixed trajectory, prepared once on the GPU as a
    voxel-major (V, C) f32 field, so that each control cycle is one coalesced
    gather (``lsdf_query_vm``) instead of a window scan.  RobotSdfBatch-like:
    ``grid``, ``n_configs``, ``d_far_global`` and a lazily transposed ``values``.
    """

    def __init__(self, traj: TrajectorySdf):
        t = N.torch()
        self.traj = traj
        self.grid = traj.grid
        self.d_far_global = traj.d_far_global
        C_ = traj.n_configs
        self.field = N.empty((self.grid.n_voxels, C_), t.float32)
        ws, _ = traj.window.device_tables()
        self._poses = R, dt, anchor = traj.config_major()  # the per-cycle link pass reads them too
        N.call("lsdf_materialize_vm", N.ptr(R), N.ptr(dt), N.ptr(anchor), C_, traj.n_links,
               traj._table, ctypes.byref(ws), ctypes.byref(self.grid.c_struct()), self.d_far_global,
               self.field, N.stream())
        self._keys = N.zeros((C_,), t.int64)  # the kernels leave it zeroed

    @property
    def n_configs(self) -> int:
        return self.traj.n_configs

    @property
    def values(self) -> np.ndarray:
        """(C, nx, ny, nz) like RobotSdfBatch.values (a transposed host copy)."""
        v = self.field.T.contiguous().cpu().numpy().reshape((self.n_configs,) + tuple(int(d) for d in self.grid.dims))
        v.flags.writeable = False
        return v

    def query_device(self, occupancy, indices_dev, n_list: int, outputs=None):
        """Enqueue one cycle: (d, link, voxel) CUDA tensors; n_list < 0 reads the
        occupied count from ``occupancy`` (a voxelized cloud's sorted list)."""
        t = N.torch()
        C_ = self.n_configs
        out = outputs if outputs is not None else {}
        if "d" not in out:
            out["d"] = N.empty((C_,), t.float32)
            out["link"] = N.empty((C_,), t.int32)
            out["voxel"] = N.empty((C_,), t.int32)
        tr = self.traj
        ws, _ = tr.window.device_tables()
        R, dt, anchor = self._poses
        N.call("lsdf_query_vm", self.field, N.ptr(R), N.ptr(dt), N.ptr(anchor), C_, tr.n_links, tr._table,
               ctypes.byref(ws), ctypes.byref(self.grid.c_struct()), N.ptr(occupancy), N.ptr(indices_dev), int(n_list),
               self.d_far_global, self._keys, out["d"], out["link"], out["voxel"], N.stream())
        return out


def _materialize(self) -> VoxelMajorSdf:
    """The voxel-major materialized field of this trajectory (prepare once, query many cycles)."""
    return VoxelMajorSdf(self)


TrajectorySdf.materialize = _materialize


# =========================================================================== reference API


def assemble_robot_sdfs(fields: Iterable, grid: EnvGrid, n_configs: int, d_far_global: float,
                        max_bytes: int = DEFAULT_BATCH_BYTES) -> RobotSdfBatch:
    """Min-merge (config, field) pairs into dense robot SDFs (query.py:61-103), on the GPU."""
    need = n_configs * grid.n_voxels * 4
    if need > max_bytes:
        raise ValidationError(
            f"robot SDF batch needs {need / 2**20:.0f} MiB for {n_configs} configurations x "
            f"{grid.n_voxels} voxels, over the {max_bytes / 2**20:.0f} MiB budget")
    t = N.torch()
    groups: dict[tuple, list] = {}
    for c, field in fields:
        if not 0 <= c < n_configs:
            raise ValidationError(f"configuration index {c} out of range")
        groups.setdefault(tuple(field.window_dims), []).append((c, field))
    out = N.empty((n_configs,) + tuple(int(d) for d in grid.dims), t.float32)
    N.call("lsdf_fill", N.ptr(out), out.numel(), float(np.float32(d_far_global)), N.stream())
    for wd, items in groups.items():
        vals = np.stack([np.ravel(f.values, order="F") for _, f in items]).astype(np.float32)
        anchors = np.stack([np.asarray(f.anchor, dtype=np.int64) for _, f in items]).astype(np.int32)
        cfg = np.asarray([c for c, _ in items], dtype=np.int32)
        N.call("lsdf_assemble", N.to_device(vals), N.to_device(anchors), N.to_device(cfg),
               len(items), N.i32x3(wd), ctypes.byref(grid.c_struct()), 0, float(d_far_global), N.ptr(out),
               N.stream())
    return RobotSdfBatch(values=out, grid=grid, d_far_global=float(d_far_global))


def _clamp_rule(d, link, voxel, clamp):
    far = d == np.float32(clamp)
    link = np.where(far, -1, link).astype(np.int32)
    voxel = np.where(far, -1, voxel).astype(np.int32)
    return link, voxel


def query_min_distances(batch, obstacles: ObstacleVoxelSet, return_stats: bool = False, *,
                        return_argmin: bool = False):
    """Minimum robot-obstacle distance per configuration (query.py:128-150).

    ``batch`` is a dense :class:`RobotSdfBatch` (gather + min kernel) or a
    :class:`TrajectorySdf` (fused direct kernel, same values).  With
    ``return_argmin`` the result is (d, link, voxel): voxel is the position in
    ``obstacles.indices`` of the first minimum, link the lowest geometry link
    attaining it (dense batches carry no link identity: -1); both are -1 when
    d equals float32(d_far_global).  ``return_stats`` reports the algorithmic
    gather count C x |occupied| (query.py:144-149).
    """
    if not batch.grid.same_geometry(obstacles.grid):
        raise GridMismatchError("obstacle set was voxelized on a different grid")
    C_ = batch.n_configs
    stats = {"gathers": int(C_ * obstacles.n_occupied)}
    clamp = np.float32(batch.d_far_global)
    if obstacles.n_occupied == 0:
        d = np.full(C_, clamp, dtype=np.float32)
        link = np.full(C_, -1, np.int32)
        voxel = np.full(C_, -1, np.int32)
    elif isinstance(batch, TrajectorySdf):
        occ, by_pos = obstacles.occupancy()
        out = batch.query_device(occ, by_pos)
        d, link, voxel = (out["d"].cpu().numpy(), out["link"].cpu().numpy(), out["voxel"].cpu().numpy())
    elif isinstance(batch, PlacedTrajectorySdf):
        out = batch.query_device(obstacles.device_indices(), obstacles.n_occupied)
        d, link, voxel = (out["d"].cpu().numpy(), out["link"].cpu().numpy(), out["voxel"].cpu().numpy())
    elif isinstance(batch, VoxelMajorSdf):
        occ, _ = obstacles.occupancy()
        out = batch.query_device(occ, obstacles.device_indices(), obstacles.n_occupied)
        d, link, voxel = (out["d"].cpu().numpy(), out["link"].cpu().numpy(), out["voxel"].cpu().numpy())
    else:
        t = N.torch()
        d_dev = N.empty((C_,), t.float32)
        a_dev = N.empty((C_,), t.int32)
        N.call("lsdf_query_dense", N.ptr(batch.device_values()), C_, ctypes.byref(batch.grid.c_struct()),
               N.ptr(obstacles.device_indices()), obstacles.n_occupied, N.ptr(d_dev), N.ptr(a_dev), N.stream())
        d = d_dev.cpu().numpy()
        link, voxel = _clamp_rule(d, np.full(C_, -1), a_dev.cpu().numpy(), clamp)
    result = (d, link, voxel) if return_argmin else d
    return (result, stats) if return_stats else result


def per_link_min_distances(fields, obstacles: ObstacleVoxelSet, n_configs: int, n_links: int,
                           d_far_global: float) -> np.ndarray:
    """Per-(configuration, link) minima from (config, link, field) triples (query.py:153-176)."""
    t = N.torch()
    out = N.empty((n_configs, n_links), t.float32)
    N.call("lsdf_fill", N.ptr(out), out.numel(), float(np.float32(d_far_global)), N.stream())
    occ, _ = obstacles.occupancy() if obstacles.n_occupied else (occupancy_workspace(obstacles.grid), False)
    if obstacles.n_occupied == 0:
        N.call("lsdf_occupancy_from_indices", None, 0, 1, ctypes.byref(obstacles.grid.c_struct()), N.ptr(occ),
               N.stream())
    groups: dict[tuple, list] = {}
    for c, li, f in fields:
        groups.setdefault(tuple(f.window_dims), []).append((c, li, f))
    for wd, items in groups.items():
        vals = np.stack([np.ravel(f.values, order="F") for *_, f in items]).astype(np.float32)
        anchors = np.stack([np.asarray(f.anchor) for *_, f in items]).astype(np.int32)
        cfg = np.asarray([c for c, _, _ in items], np.int32)
        lnk = np.asarray([li for _, li, _ in items], np.int32)
        dfar = np.asarray([np.float32(f.d_far) for *_, f in items], np.float32)
        N.call("lsdf_per_link_fields", N.to_device(vals), N.to_device(anchors),
               N.to_device(cfg), N.to_device(lnk), N.to_device(dfar), len(items),
               N.i32x3(wd), n_links, ctypes.byref(obstacles.grid.c_struct()), N.ptr(occ), N.ptr(out), N.stream())
    return out.cpu().numpy()


def stream_min_distances(batch, frames: Iterable) -> Iterator[tuple[float, np.ndarray]]:
    """Per-cycle distance vectors for (timestamp, points) frames (query.py:294-306)."""
    for timestamp, points in frames:
        yield timestamp, query_min_distances(batch, voxelize_pointcloud(points, batch.grid))


def query_trajectory(robot, configs, sdfs, grid: EnvGrid, provider_or_window, points=None, *,
                     obstacles: ObstacleVoxelSet | None = None, d_far_global=None):
    """Configurations + points (or voxels) -> (d f32[C], link i32[C], voxel i32[C]).

    ``link`` indexes the geometry links (``robot.geometry_links``); ``voxel``
    is the position in the sorted occupied-voxel list.
    """
    from .placement import ExactTransformProvider, WindowGeometry

    window = getattr(provider_or_window, "window", provider_or_window)
    if isinstance(provider_or_window, (WindowGeometry, ExactTransformProvider)):
        traj = TrajectorySdf.from_configs(robot, configs, sdfs, grid, window, d_far_global)
    else:  # another provider (neural): its placement, never silently the exact transform
        from .robot import ConfigBatch, LinkPoseBatch, forward_kinematics_batch

        poses = forward_kinematics_batch(robot, configs if isinstance(configs, ConfigBatch) else ConfigBatch(configs))
        gl = robot.geometry_links
        geo = LinkPoseBatch(rotations=poses.rotations[:, gl], translations=poses.translations[:, gl])
        traj = PlacedTrajectorySdf.from_poses(sdfs, geo, grid, provider_or_window, d_far_global)
    obs = obstacles if obstacles is not None else voxelize_pointcloud(points, grid)
    return query_min_distances(traj, obs, return_argmin=True)


# =========================================================================== sphere baseline


@dataclass(frozen=True, eq=False)
class SphereRobotModel:
    """Per-link covering spheres in link frames (query.py:179-212), flattened:
    sphere k belongs to link ``link_indices[k]``."""

    link_indices: np.ndarray
    centers: np.ndarray
    radii: np.ndarray

    def __post_init__(self):
        if (np.asarray(self.radii) <= 0).any():
            raise ValidationError("sphere radii must be positive")

    @property
    def n_spheres(self) -> int:
        return len(self.radii)

    @classmethod
    def from_robot(cls, model) -> "SphereRobotModel":
        """Flatten the robot JSON's ``spheres`` section, link by link in its order."""
        flat = [(model.link_index(name), c, r) for name, entries in model.sphere_model.items() for c, r in entries]
        if not flat:
            raise ValidationError(f"robot {model.name} declares no spheres")
        idx, centers, radii = zip(*flat)
        return cls(link_indices=np.int64(idx), centers=np.float64(centers), radii=np.float64(radii))


def validate_sphere_model(model, spheres: SphereRobotModel, rng: np.random.Generator, n_samples: int = 2048,
                          tol: float = 1e-9) -> float:
    """Worst excess of a link's surface samples over its covering spheres
    (query.py:215-251); host-side, consumes ``rng`` like the reference
    (links in order, n_samples per link).  Raises past ``tol``."""
    worst = -np.inf
    for li, link in enumerate(model.links):
        geom = link.geometry
        if geom is None:
            continue
        own = np.flatnonzero(spheres.link_indices == li)
        if own.size == 0:
            raise ValidationError(f"link {link.name} has geometry but no spheres")
        samples = (geom.sample_surface(n_samples, rng) if isinstance(geom, TriangleMesh)
                   else primitive_surface_points(geom, n_samples, rng))
        gaps = np.linalg.norm(samples[:, None, :] - spheres.centers[own][None], axis=-1) - spheres.radii[own]
        worst = max(worst, float(gaps.min(axis=1).max()))
        if worst > tol:
            raise ValidationError(f"link {link.name}: surface escapes the covering spheres by {worst:.2e} m")
    return worst


def sphere_baseline_distances(spheres: SphereRobotModel, poses, obstacles: ObstacleVoxelSet, grid: EnvGrid,
                              chunk: int = 64, return_stats: bool = False):
    """Covering-sphere comparator (query.py:254-291), evaluated on the GPU in fp64."""
    if not grid.same_geometry(obstacles.grid):
        raise GridMismatchError("obstacle set was voxelized on a different grid")
    C_ = poses.n_configs
    if obstacles.n_occupied == 0:
        d = np.full(C_, np.inf, dtype=np.float64)
        return (d, {"distance_evals": 0}) if return_stats else d
    t = N.torch()
    L = poses.n_links
    R = N.to_device(np.ascontiguousarray(poses.rotations, dtype=np.float64), t.float64)
    T = N.to_device(np.ascontiguousarray(poses.translations, dtype=np.float64), t.float64)
    out = N.empty((C_,), t.float64)
    N.call("lsdf_sphere_baseline", N.ptr(R), N.ptr(T), C_, L,
           N.to_device(spheres.link_indices.astype(np.int32)),
           N.to_device(np.ascontiguousarray(spheres.centers, dtype=np.float64)),
           N.to_device(np.ascontiguousarray(spheres.radii, dtype=np.float64)), spheres.n_spheres,
           N.ptr(obstacles.device_indices()), obstacles.n_occupied, ctypes.byref(grid.c_struct()), N.ptr(out),
           N.stream())
    d = out.cpu().numpy()
    if return_stats:
        return d, {"distance_evals": int(C_ * spheres.n_spheres * obstacles.n_occupied)}
    return d


# =========================================================================== frame IO (host plumbing)


_FRAME_COUNT = struct.Struct("<I")


def write_pointcloud_frame(path, points) -> None:
    """Frame file (query.py:313-318): uint32 point count, then xyz as little-endian f32."""
    pts = np.ascontiguousarray(np.asarray(points, dtype="<f4").reshape(-1, 3))
    Path(path).write_bytes(_FRAME_COUNT.pack(len(pts)) + pts.tobytes())


def read_pointcloud_frame(path) -> np.ndarray:
    """(N, 3) f64 points of a frame file; ValidationError when the data is short."""
    data = Path(path).read_bytes()
    (count,) = _FRAME_COUNT.unpack_from(data)
    avail = (len(data) - _FRAME_COUNT.size) // 4
    if avail < 3 * count:
        raise ValidationError(f"{path}: truncated point data")
    return np.frombuffer(data, dtype="<f4", count=3 * count, offset=_FRAME_COUNT.size).reshape(count, 3) \
        .astype(np.float64)


def read_cloud_manifest(path) -> list[tuple[float, Path]]:
    """Manifest: one ``<timestamp_ms> <frame file>`` per line, paths relative to
    the manifest; blank lines and ``#`` comments skipped (query.py:330-341)."""
    base = Path(path).parent
    entries = (ln.strip() for ln in Path(path).read_text().splitlines())
    pairs = (ln.split(maxsplit=1) for ln in entries if ln and not ln.startswith("#"))
    return [(float(stamp), base / name) for stamp, name in pairs]


def iter_cloud_frames(manifest_path) -> Iterator[tuple[float, np.ndarray]]:
    return ((stamp, read_pointcloud_frame(p)) for stamp, p in read_cloud_manifest(manifest_path))


def write_distance_csv(path, rows, n_configs: int) -> None:
    """timestamp_ms,d_0..d_{C-1} header, one row per cycle (%.3f stamp, %.6f distances)."""
    lines = [",".join(["timestamp_ms", *(f"d_{i}" for i in range(n_configs))])]
    lines += [",".join([f"{stamp:.3f}", *(f"{d:.6f}" for d in dists)]) for stamp, dists in rows]
    Path(path).write_text("".join(line + "\n" for line in lines))
