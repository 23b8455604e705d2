"""DistanceChecker — the real-time entry point: configurations + cloud → (d, link, voxel).

One object per (robot, link SDFs, environment grid, window).  ``prepare``
sizes device buffers and pinned host staging for a batch shape and captures
the whole control-cycle step in one CUDA graph:

    H2D(q, points) → fk_align → voxelize (memset, scatter, rank) →
    query_direct (lookup + min/argmin, finished in-kernel) → D2H(d, link, voxel, flags)

so a 500-waypoint query is a single graph launch plus one stream sync.  The
point capacity is fixed per capture; shorter clouds are padded with NaN,
which the voxelizer drops exactly like out-of-grid points (query.py:112).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .errors import LimitViolationError, NoOverlapError, ValidationError
from .query import TrajectorySdf, occupancy_workspace, voxelize_device
from .robot import fk_device


class DistanceChecker:
    def __init__(self, robot, sdfs, grid, window, *, d_far_global=None, check_limits: bool = True):
        from .placement import _check_links

        self.robot = robot
        self.sdfs = list(sdfs)
        if len(self.sdfs) != len(robot.geometry_links):
            raise ValidationError(f"{len(self.sdfs)} SDFs for {len(robot.geometry_links)} geometry links")
        self.grid = grid
        self.window = getattr(window, "window", window)
        _check_links(self.sdfs, self.window)
        self.d_far_global = float(min(s.d_far for s in self.sdfs) if d_far_global is None else d_far_global)
        self.check_limits = check_limits
        self._limits = robot.position_limits()
        self._shape = None
        self._graph = None
        self._graph_dev = None

    # ------------------------------------------------------------------ buffers
    def prepare(self, n_configs: int, n_points: int, points_dtype=np.float32, use_graph: bool = True):
        t = N.torch()
        dev = N.device()
        tdt = t.float32 if np.dtype(points_dtype) == np.float32 else t.float64
        C_, D = int(n_configs), self.robot.dof
        self._shape = (C_, int(n_points), np.dtype(points_dtype))
        self.q_host = t.empty((C_, D), dtype=t.float64, pin_memory=True)
        self.p_host = t.full((int(n_points), 3), float("nan"), dtype=tdt, pin_memory=True)
        self.q_dev = t.zeros((C_, D), dtype=t.float64, device=dev)
        self.p_dev = t.full((int(n_points), 3), float("nan"), dtype=tdt, device=dev)
        self.ws = occupancy_workspace(self.grid)
        self.fk_out = {}
        fk_device(self.robot, self.q_dev, all_links=False, grid=self.grid, window_dims=self.window.dims,
                  outputs=self.fk_out)  # allocates outputs (values are garbage until run)
        self.traj = TrajectorySdf(self.sdfs, self.grid, self.window, self.fk_out["R_geo"], self.fk_out["dt_geo"],
                                  self.fk_out["anchor_geo"], self.d_far_global)
        self.q_out = {}
        self.traj.query_device(self.ws, False, outputs=self.q_out)
        self.d_host = t.empty((C_,), dtype=t.float32, pin_memory=True)
        self.link_host = t.empty((C_,), dtype=t.int32, pin_memory=True)
        self.voxel_host = t.empty((C_,), dtype=t.int32, pin_memory=True)
        self.flags_host = t.empty((4,), dtype=t.int32, pin_memory=True)
        self.window.device_tables()
        for sdf in self.sdfs:
            sdf.packed_values()
        self._side = t.cuda.Stream()
        t.cuda.synchronize()
        if use_graph:
            self._capture()
        return self

    def host_inputs(self):
        """Pinned numpy views (configs (C, D) f64, points (N, 3)) the caller may fill in place."""
        return self.q_host.numpy(), self.p_host.numpy()

    # ------------------------------------------------------------------ the step
    # FK+alignment and voxelization are independent: FK runs on a side stream
    # while the cloud is voxelized, the query joins both (two graph branches).
    def _fk(self, h2d: bool):
        if h2d:
            self.q_dev.copy_(self.q_host, non_blocking=True)
        self.fk_out["flags"].zero_()
        fk_device(self.robot, self.q_dev, all_links=False, grid=self.grid, window_dims=self.window.dims,
                  outputs=self.fk_out)

    def _run(self, h2d: bool):
        t = N.torch()
        main = t.cuda.current_stream()
        self._side.wait_stream(main)
        with t.cuda.stream(self._side):
            self._fk(h2d)
        if h2d:
            self.p_dev.copy_(self.p_host, non_blocking=True)
        voxelize_device(self.p_dev, self.grid, workspace=self.ws)
        main.wait_stream(self._side)
        self.traj.query_device(self.ws, False, outputs=self.q_out)
        if h2d:
            self.d_host.copy_(self.q_out["d"], non_blocking=True)
            self.link_host.copy_(self.q_out["link"], non_blocking=True)
            self.voxel_host.copy_(self.q_out["voxel"], non_blocking=True)
            self.flags_host.copy_(self.fk_out["flags"], non_blocking=True)

    def _compute(self):
        """Device work of one cycle (inputs already in q_dev / p_dev)."""
        self._run(False)

    def _step(self):
        """H2D of the inputs, the cycle, D2H of (d, link, voxel, flags)."""
        self._run(True)

    def _capture(self):
        t = N.torch()
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            for _ in range(2):  # warm-up outside capture (sets kernel attributes, pools)
                self._step()
        t.cuda.current_stream().wait_stream(s)
        t.cuda.synchronize()
        self._graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self._graph):
            self._step()
        self._graph_dev = t.cuda.CUDAGraph()
        with t.cuda.graph(self._graph_dev):
            self._compute()
        t.cuda.synchronize()

    # ------------------------------------------------------------------ public calls
    def launch(self, device_only: bool = False):
        """Enqueue one cycle (graph replay when captured); no synchronisation."""
        g = self._graph_dev if device_only else self._graph
        if g is not None:
            g.replay()
        elif device_only:
            self._compute()
        else:
            self._step()

    def query(self, configs=None, points=None):
        """One control cycle from host arrays; returns numpy (d, link, voxel)."""
        if self._shape is None:
            raise ValidationError("call prepare(n_configs, n_points) first")
        C_, cap, _ = self._shape
        q_np, p_np = self.host_inputs()
        if configs is not None:
            q = np.asarray(configs, dtype=np.float64)
            if q.shape != q_np.shape:
                raise ValidationError(f"configurations {q.shape} do not match the prepared {q_np.shape}")
            q_np[...] = q
        if points is not None:
            p = np.asarray(points).reshape(-1, 3)
            if len(p) > cap:
                raise ValidationError(f"{len(p)} points exceed the prepared capacity {cap}")
            p_np[: len(p)] = p
            p_np[len(p):] = np.nan
        self.launch()
        N.torch().cuda.current_stream().synchronize()
        self._raise_flags(q_np)
        return self.d_host.numpy().copy(), self.link_host.numpy().copy(), self.voxel_host.numpy().copy()

    def _raise_flags(self, q_np):
        f = self.flags_host.numpy()
        if self.check_limits and f[0]:
            lim = self._limits
            bad = (q_np < lim[:, 0]) | (q_np > lim[:, 1])
            cs, js = np.nonzero(bad)
            raise LimitViolationError(list(zip(cs.tolist(), js.tolist())))
        if f[1]:
            raise NoOverlapError(f"{int(f[1])} window(s) miss the grid entirely")
