"""DistanceChecker — the real-time entry point: configurations + cloud → (d, link, voxel).

One object per (robot, link SDFs, environment grid, window).  ``prepare``
sizes device buffers and pinned host buffers for a batch shape and captures
one control cycle as a CUDA graph with two branches:

    side stream:    fk_align (reads the configurations)  ──┐
    main stream:    voxelize bitmap (memset, scatter)   ──┴─> query scan ──┬─> finalize ──> (d, link, voxel)
    prefix stream:                   └─> rank prefix ───────────────────────┘

End to end (``query``) the kernels read the configurations and the cloud
straight from page-locked host memory and the query writes (d, link, voxel)
straight back to page-locked host memory (zero-copy over PCIe, mapped by
``lsdf_host_device_pointer``), so the transfer overlaps the voxelization
instead of preceding it; when mapping is unavailable the graph stages the
same bytes with explicit async copies.  ``launch(device_only=True)`` replays
the same cycle on device-resident inputs (the bench's HBM-resident number).

The point capacity is fixed per capture; shorter clouds are padded with NaN,
which the voxelizer drops exactly like out-of-grid points (query.py:112).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .errors import LimitViolationError, NoOverlapError, ValidationError
from .query import TrajectorySdf, occupancy_workspace

# batch size from which FK runs one thread per configuration (lsdf_fk.cu
# FK_SERIAL_MIN) and the checker keeps its poses link-major
LINK_MAJOR_MIN = 6144
DENSE_HINT_POINTS = 65536  # clouds from this capacity set LSDF_QUERY_DENSE_HINT (config 2: 100k; config 5: 30k)


def _require_exact(window_or_provider, who: str):
    """The fused real-time cycle evaluates the exact transform; refuse another
    provider loudly instead of silently using its window with exact values."""
    from .placement import ExactTransformProvider, WindowGeometry

    if isinstance(window_or_provider, (WindowGeometry, ExactTransformProvider)):
        return
    raise ValidationError(f"{who} runs the exact transform (placement.py:148-169) in its fused cycle; for "
                          f"{type(window_or_provider).__name__} use TrajectorySdf.from_poses(..., provider) or "
                          f"MaterializedChecker(..., provider)")


class DistanceChecker:
    def __init__(self, robot, sdfs, grid, window, *, d_far_global=None, check_limits: bool = True):
        from .placement import _check_links

        self.robot = robot
        self.sdfs = list(sdfs)
        if len(self.sdfs) != len(robot.geometry_links):
            raise ValidationError(f"{len(self.sdfs)} SDFs for {len(robot.geometry_links)} geometry links")
        self.grid = grid
        _require_exact(window, "DistanceChecker")
        self.window = getattr(window, "window", window)
        _check_links(self.sdfs, self.window)
        self.d_far_global = float(min(s.d_far for s in self.sdfs) if d_far_global is None else d_far_global)
        self.check_limits = check_limits
        self._limits = robot.position_limits()
        self._shape = None
        self._graph = None
        self._graph_dev = None

    # ------------------------------------------------------------------ buffers
    def prepare(self, n_configs: int, n_points: int, points_dtype=np.float32, use_graph: bool = True,
                zero_copy: bool = True, contiguous_inputs: bool = False):
        """Size buffers for (n_configs, n_points) and capture the cycle graphs.

        contiguous_inputs: configurations and cloud share one pinned host
        buffer and one device buffer (``in_host`` / ``in_dev``), so a pipeline
        moves a cycle's inputs with a single copy-engine transfer.
        """
        t = N.torch()
        dev = N.device()
        pdt = np.dtype(points_dtype)
        if pdt not in (np.float32, np.float64):
            raise ValidationError(f"points must be float32 or float64, got {pdt}")
        tdt = t.float32 if pdt == np.float32 else t.float64
        C_, D, G = int(n_configs), self.robot.dof, len(self.sdfs)
        P = int(n_points)
        self._shape = (C_, P, pdt)
        pin = dict(pin_memory=True)
        # host side (page-locked)
        if contiguous_inputs:  # [configs f64 | pad to 256 B | points]: one transfer per cycle
            q_bytes = (C_ * D * 8 + 255) // 256 * 256
            nbytes = q_bytes + P * 3 * pdt.itemsize
            self.in_host = t.empty((nbytes,), dtype=t.uint8, **pin)
            self.in_dev = t.empty((nbytes,), dtype=t.uint8, device=dev)
            self.q_host = self.in_host[: C_ * D * 8].view(t.float64).view(C_, D)
            self.p_host = self.in_host[q_bytes:].view(tdt).view(P, 3)
            self.q_host.zero_()
            self.p_host.fill_(float("nan"))
        else:
            self.in_host = self.in_dev = None
            self.q_host = t.zeros((C_, D), dtype=t.float64, **pin)
            self.p_host = t.full((P, 3), float("nan"), dtype=tdt, **pin)
        self.d_host = t.zeros((C_,), dtype=t.float32, **pin)
        self.link_host = t.zeros((C_,), dtype=t.int32, **pin)
        self.voxel_host = t.zeros((C_,), dtype=t.int32, **pin)
        self.flags_host = t.zeros((4,), dtype=t.int32, **pin)
        self._np = {k: getattr(self, k + "_host").numpy() for k in ("q", "p", "d", "link", "voxel", "flags")}
        # device side
        if contiguous_inputs:
            self.q_dev = self.in_dev[: C_ * D * 8].view(t.float64).view(C_, D)
            self.p_dev = self.in_dev[q_bytes:].view(tdt).view(P, 3)
            self.q_dev.zero_()
            self.p_dev.fill_(float("nan"))
        else:
            self.q_dev = t.zeros((C_, D), dtype=t.float64, device=dev)
            self.p_dev = t.full((P, 3), float("nan"), dtype=tdt, device=dev)
        # large batches keep the poses link-major ((G, C, .) storage, exposed as
        # (C, G, .) views): FK then writes each link's records contiguously
        self.link_major = C_ >= LINK_MAJOR_MIN
        if self.link_major:
            self.R_geo = t.zeros((G, C_, 3, 3), dtype=t.float64, device=dev).transpose(0, 1)
            self.dt_geo = t.zeros((G, C_, 3), dtype=t.float64, device=dev).transpose(0, 1)
            self.anchor_geo = t.zeros((G, C_, 3), dtype=t.int32, device=dev).transpose(0, 1)
        else:
            self.R_geo = t.zeros((C_, G, 3, 3), dtype=t.float64, device=dev)
            self.dt_geo = t.zeros((C_, G, 3), dtype=t.float64, device=dev)
            self.anchor_geo = t.zeros((C_, G, 3), dtype=t.int32, device=dev)
        self._fk_entry = "lsdf_fk_align_link_major" if self.link_major else "lsdf_fk_align"
        # self-resetting FK flags: no reset node ahead of FK on the cycle's critical branch
        self._fk_opts = (N.FK_LINK_MAJOR if self.link_major else 0) | N.FK_FLAGS_SELF_RESET
        self._qflags = N.QUERY_POSES_LINK_MAJOR if self.link_major else 0
        if n_points >= DENSE_HINT_POINTS:  # dense obstacles: the one-wave latency walk (lsdf_query.cu)
            self._qflags |= N.QUERY_DENSE_HINT
        # FK flags: [0..1] published per cycle, [2..4] the kernel's self-resetting counters
        self.flags = t.zeros((8,), dtype=t.int32, device=dev)
        self.limits = N.to_device(np.ascontiguousarray(self._limits), t.float64)
        self.d_dev = t.zeros((C_,), dtype=t.float32, device=dev)
        self.link_dev = t.zeros((C_,), dtype=t.int32, device=dev)
        self.voxel_dev = t.zeros((C_,), dtype=t.int32, device=dev)
        self.ws = occupancy_workspace(self.grid)
        self.traj = TrajectorySdf(self.sdfs, self.grid, self.window, self.R_geo, self.dt_geo, self.anchor_geo,
                                  self.d_far_global, link_major=self.link_major)
        self.qws = t.zeros((int(N.lib().lsdf_query_workspace_bytes(C_, G)),), dtype=t.uint8, device=dev)
        self._wstruct, _ = self.window.device_tables()
        for sdf in self.sdfs:
            sdf.packed_values()
        # mapped addresses for the zero-copy end-to-end cycle
        self._map = None
        if zero_copy:
            try:
                self._map = {k: N.mapped_pointer(getattr(self, k + "_host")) for k in ("q", "p", "d", "link", "voxel")}
            except Exception:  # mapping unavailable: the graph stages copies instead
                self._map = None
        self._side = t.cuda.Stream()
        self._prefix_stream = t.cuda.Stream()
        self._env = ctypes.byref(self.grid.c_struct())
        self._W = N.i32x3(self.window.dims)
        self._chain = self.robot.chain_table()
        t.cuda.synchronize()
        if use_graph:
            self._capture()
        return self

    def host_inputs(self):
        """Pinned numpy views (configs (C, D) f64, points (N, 3)) the caller may fill in place."""
        return self._np["q"], self._np["p"]

    @property
    def zero_copy(self) -> bool:
        return self._map is not None

    # ------------------------------------------------------------------ the cycle
    def _run(self, e2e: bool):
        t = N.torch()
        C_, P, pdt = self._shape
        main = t.cuda.current_stream()
        side = self._side
        zc = e2e and self._map is not None
        staged = e2e and self._map is None
        side.wait_stream(main)
        with t.cuda.stream(side):
            if staged:
                self.q_dev.copy_(self.q_host, non_blocking=True)
            q_ptr = self._map["q"] if zc else N.ptr(self.q_dev)
            N.call("lsdf_fk_align_ex", self._chain, self.robot.n_links, len(self.sdfs), q_ptr, C_, self.robot.dof,
                   N.ptr(self.limits), self._env, self._W, None, None, N.ptr(self.R_geo), N.ptr(self.dt_geo),
                   N.ptr(self.anchor_geo), N.ptr(self.flags), self._fk_opts, side.cuda_stream)
        if staged:
            self.p_dev.copy_(self.p_host, non_blocking=True)
        p_ptr = self._map["p"] if zc else N.ptr(self.p_dev)
        # the rank prefix is only needed by the finalize: it runs on a third
        # stream while the scan (which needs the bitmap alone) runs
        N.call("lsdf_voxelize_bitmap", p_ptr, int(pdt == np.float32), P, self._env, N.ptr(self.ws),
               main.cuda_stream)
        pre = self._prefix_stream
        pre.wait_stream(main)
        N.call("lsdf_occupancy_prefix", self._env, N.ptr(self.ws), pre.cuda_stream)
        main.wait_stream(side)
        if e2e:
            with t.cuda.stream(side):  # 16 B of flags back to the host, off the critical path
                self.flags_host.copy_(self.flags[:4], non_blocking=True)
        if zc:
            outs = (self._map["d"], self._map["link"], self._map["voxel"])
        else:
            outs = (N.ptr(self.d_dev), N.ptr(self.link_dev), N.ptr(self.voxel_dev))
        tr = self.traj
        args = (N.ptr(self.R_geo), N.ptr(self.dt_geo), N.ptr(self.anchor_geo), C_, tr.n_links, tr._table,
                ctypes.byref(self._wstruct), self._env, N.ptr(self.ws), self._qflags,
                self.d_far_global, N.ptr(self.qws),
                outs[0], outs[1], outs[2], None, main.cuda_stream)
        N.call("lsdf_query_scan", *args)
        main.wait_stream(pre)
        N.call("lsdf_query_finalize", *args)
        if staged:
            self.d_host.copy_(self.d_dev, non_blocking=True)
            self.link_host.copy_(self.link_dev, non_blocking=True)
            self.voxel_host.copy_(self.voxel_dev, non_blocking=True)
        if e2e:
            main.wait_stream(side)

    def _capture(self):
        t = N.torch()
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            for _ in range(2):  # warm-up outside capture (kernel attributes, allocator pools)
                self._run(True)
                self._run(False)
        t.cuda.current_stream().wait_stream(s)
        t.cuda.synchronize()
        self._graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self._graph):
            self._run(True)
        self._graph_dev = t.cuda.CUDAGraph()
        with t.cuda.graph(self._graph_dev):
            self._run(False)
        t.cuda.synchronize()

    # ------------------------------------------------------------------ public calls
    def launch(self, device_only: bool = False):
        """Enqueue one cycle (graph replay when captured); no synchronisation.

        device_only: inputs from q_dev / p_dev, results to d_dev / link_dev / voxel_dev.
        """
        g = self._graph_dev if device_only else self._graph
        if g is not None:
            g.replay()
        else:
            self._run(not device_only)

    def query(self, configs=None, points=None):
        """One control cycle from host arrays; returns numpy (d, link, voxel)."""
        if self._shape is None:
            raise ValidationError("call prepare(n_configs, n_points) first")
        C_, cap, _ = self._shape
        q_np, p_np = self._np["q"], self._np["p"]
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
        f = self._np["flags"]
        if f[0] or f[1]:
            self._raise_flags(q_np, f)
        return self._np["d"].copy(), self._np["link"].copy(), self._np["voxel"].copy()

    def _raise_flags(self, q_np, f):
        if self.check_limits and f[0]:
            lim = self._limits
            bad = (q_np < lim[:, 0]) | (q_np > lim[:, 1])
            cs, js = np.nonzero(bad)
            raise LimitViolationError(list(zip(cs.tolist(), js.tolist())))
        if f[1]:
            raise NoOverlapError(f"{int(f[1])} window(s) miss the grid entirely")


class _CycleResults:
    """Outcome bookkeeping shared by the pipelines: a recycled slot is drained
    into ``_done`` (copies plus any flag error) and each ticket's result(),
    including its error, is delivered by that ticket's own result() call."""

    def _drain(self, s):
        """Wait for the slot's cycle and keep its outcome (copies, and any limit /
        no-overlap error) for its own result(ticket) call, so recycling the slot
        neither raises an older cycle's error here nor drops its distances."""
        s["ev"]["d2h"].synchronize()
        d, link, voxel, flags = (a.numpy() for a in s["out"])
        err = None
        if flags[0] or flags[1]:
            chk = s["chk"]
            try:
                chk._raise_flags(chk.host_inputs()[0], flags)
            except Exception as exc:  # noqa: BLE001 — re-raised from result(ticket)
                err = exc
        self._done[s["ticket"]] = (d.copy(), link.copy(), voxel.copy(), err)
        for old in [k for k in self._done if k < self._next - 4 * len(self.slots)]:
            del self._done[old]
        s["busy"] = False

    def result(self, ticket: int):
        """(d, link, voxel) numpy copies of a submitted cycle (blocks until it is
        back on the host); raises that cycle's LimitViolationError /
        NoOverlapError, if any."""
        s = self._slot(ticket)
        if s["ticket"] == ticket and s["busy"]:
            self._drain(s)
        if ticket not in self._done:
            raise ValidationError(f"cycle {ticket} is no longer held (pipeline depth {self.depth})")
        d, link, voxel, err = self._done.pop(ticket)
        if err is not None:
            raise err
        return d, link, voxel



class CheckerPipeline(_CycleResults):
    """Throughput form of DistanceChecker: ``depth`` cycles in flight.

    Each slot is a prepared DistanceChecker (its own device buffers and
    device-input graph) plus page-locked host buffers.  A cycle is three
    stream-ordered pieces:

        copy stream:    H2D configurations + cloud of slot s (copy engine)
        compute stream: the slot's graph (fk_align || voxelize -> query)
        d2h stream:     (d, link, voxel) + FK flags of slot s back to the host

    so the PCIe transfers of cycle i+1 and the read-back of cycle i-1 run on
    the copy engines while cycle i computes (zero-copy reads, as used by the
    latency path, would need SMs the persistent query kernel occupies).
    Producers write the next cycle's inputs straight into ``inputs()`` (pinned
    numpy views), then ``submit()``; ``result(ticket)`` waits for that cycle.
    """

    def __init__(self, robot, sdfs, grid, window, n_configs: int, n_points: int, points_dtype=np.float32,
                 depth: int = 2, **kw):
        t = N.torch()
        if depth < 1:
            raise ValidationError("pipeline depth must be >= 1")
        self.slots = []
        for _ in range(depth):
            chk = DistanceChecker(robot, sdfs, grid, window, **kw).prepare(n_configs, n_points, points_dtype,
                                                                           zero_copy=False, contiguous_inputs=True)
            pin = dict(pin_memory=True)
            host_out = (t.zeros((n_configs,), dtype=t.float32, **pin), t.zeros((n_configs,), dtype=t.int32, **pin),
                        t.zeros((n_configs,), dtype=t.int32, **pin), t.zeros((4,), dtype=t.int32, **pin))
            ev = {k: t.cuda.Event() for k in ("h2d", "compute", "d2h")}
            self.slots.append({"chk": chk, "out": host_out, "ev": ev, "busy": False, "ticket": -1})
        self.copy = t.cuda.Stream()
        self.compute = t.cuda.Stream()
        self.d2h = t.cuda.Stream()
        self._next = 0
        self._done = {}  # ticket -> (d, link, voxel, error) of cycles drained before their result() call

    @property
    def depth(self) -> int:
        return len(self.slots)

    def _slot(self, ticket):
        return self.slots[ticket % len(self.slots)]

    def inputs(self):
        """Pinned (configs, points) views of the next cycle's slot (waits if it is still in flight)."""
        s = self._slot(self._next)
        if s["busy"]:
            self._drain(s)
        return s["chk"].host_inputs()

    def submit(self, configs=None, points=None) -> int:
        """Enqueue the next cycle; optional arrays are copied into the slot's pinned inputs first."""
        t = N.torch()
        ticket = self._next
        s = self._slot(ticket)
        if s["busy"]:
            self._drain(s)
        chk = s["chk"]
        q_np, p_np = chk.host_inputs()
        if configs is not None:
            q_np[...] = np.asarray(configs, dtype=np.float64)
        if points is not None:
            p = np.asarray(points).reshape(-1, 3)
            if len(p) > len(p_np):
                raise ValidationError(f"{len(p)} points exceed the prepared capacity {len(p_np)}")
            p_np[: len(p)] = p
            p_np[len(p):] = np.nan
        ev = s["ev"]
        with t.cuda.stream(self.copy):
            self.copy.wait_event(ev["compute"])  # the slot's device inputs are free again
            chk.in_dev.copy_(chk.in_host, non_blocking=True)  # configurations + cloud, one transfer
            ev["h2d"].record(self.copy)
        with t.cuda.stream(self.compute):
            self.compute.wait_event(ev["h2d"])
            self.compute.wait_event(ev["d2h"])  # the previous results of this slot were read back
            chk.launch(device_only=True)
            ev["compute"].record(self.compute)
        d, link, voxel, flags = s["out"]
        with t.cuda.stream(self.d2h):
            self.d2h.wait_event(ev["compute"])
            d.copy_(chk.d_dev, non_blocking=True)
            link.copy_(chk.link_dev, non_blocking=True)
            voxel.copy_(chk.voxel_dev, non_blocking=True)
            flags.copy_(chk.flags[:4], non_blocking=True)
            ev["d2h"].record(self.d2h)
        s["busy"], s["ticket"] = True, ticket
        self._next += 1
        return ticket

class MaterializedChecker:
    """The paper's two-phase use for a FIXED trajectory:
    the robot SDF is prepared once as a voxel-major field (``VoxelMajorSdf``),
    then every control cycle is one CUDA graph — voxelize the frame (read
    zero-copy from pinned memory, with the sorted occupied list) and one
    coalesced gather + the exact argmin-link pass, results written back to
    pinned memory.  Same (d, link, voxel) as DistanceChecker on the same
    trajectory (tests/test_gpu_parity.py::test_materialized_checker).
    """

    def __init__(self, robot, sdfs, grid, window, configs, *, d_far_global=None):
        """``window``: a WindowGeometry / ExactTransformProvider (the voxel-major
        field, one CUDA graph per cycle), or another TransformProvider such as
        NeuralTransformProvider — the trajectory's windows are then placed with
        that provider once (PlacedTrajectorySdf) and each cycle is the dense
        gather + Appendix-B link (not graph-captured: the occupied count sizes
        the gather)."""
        from .placement import ExactTransformProvider, WindowGeometry, place_windows_device
        from .query import PlacedTrajectorySdf, TrajectorySdf

        self.grid = grid
        geom = getattr(window, "window", window)
        self.traj = TrajectorySdf.from_configs(robot, configs, sdfs, grid, geom, d_far_global)
        self.provider = None if isinstance(window, (WindowGeometry, ExactTransformProvider)) else window
        if self.provider is None:
            self.field = self.traj.materialize()
        else:
            R, dt, anchor = self.traj.config_major()
            win = place_windows_device(self.traj.sdfs, R, dt, geom, self.provider)
            self.field = PlacedTrajectorySdf(self.traj.sdfs, grid, geom, win, anchor, self.traj.d_far_global,
                                             self.provider)
        self._graph = None

    def prepare(self, n_points: int, points_dtype=np.float32, use_graph: bool = True):
        t = N.torch()
        pdt = np.dtype(points_dtype)
        if pdt not in (np.float32, np.float64):
            raise ValidationError(f"points must be float32 or float64, got {pdt}")
        tdt = t.float32 if pdt == np.float32 else t.float64
        C_ = self.traj.n_configs
        self._n, self._pdt = int(n_points), pdt
        pin = dict(pin_memory=True)
        self.p_host = t.full((self._n, 3), float("nan"), dtype=tdt, **pin)
        self.out_host = {"d": t.zeros((C_,), dtype=t.float32, **pin), "link": t.zeros((C_,), dtype=t.int32, **pin),
                         "voxel": t.zeros((C_,), dtype=t.int32, **pin)}
        if self.provider is not None:  # placed windows: an un-captured cycle (see __init__)
            return self
        self._p_ptr = N.mapped_pointer(self.p_host)
        self._outs = {k: v for k, v in self.out_host.items()}
        self.occ = occupancy_workspace(self.grid)
        self.idx = N.empty((self.grid.n_voxels, 3), t.int32)
        self._env = ctypes.byref(self.grid.c_struct())
        self._d = N.empty((C_,), t.float32)
        self._l = N.empty((C_,), t.int32)
        self._v = N.empty((C_,), t.int32)
        t.cuda.synchronize()
        if use_graph:
            s = t.cuda.Stream()
            s.wait_stream(t.cuda.current_stream())
            with t.cuda.stream(s):
                for _ in range(2):
                    self._run()
            t.cuda.current_stream().wait_stream(s)
            t.cuda.synchronize()
            self._graph = t.cuda.CUDAGraph()
            with t.cuda.graph(self._graph):
                self._run()
            t.cuda.synchronize()
        return self

    def _run(self):
        t = N.torch()
        N.call("lsdf_voxelize", self._p_ptr, int(self._pdt == np.float32), self._n, self._env, N.ptr(self.occ),
               N.ptr(self.idx), t.cuda.current_stream().cuda_stream)
        out = {"d": self._d, "link": self._l, "voxel": self._v}
        self.field.query_device(self.occ, self.idx, -1, outputs=out)
        for k in ("d", "link", "voxel"):
            self.out_host[k].copy_(out[k], non_blocking=True)

    def host_points(self):
        """The pinned (n_points, 3) buffer a producer may fill in place."""
        return self.p_host.numpy()

    def query(self, points=None):
        """One cycle from host points; returns numpy (d, link, voxel)."""
        t = N.torch()
        if points is not None:
            p = np.asarray(points).reshape(-1, 3)
            if len(p) > self._n:
                raise ValidationError(f"{len(p)} points exceed the prepared capacity {self._n}")
            host = self.p_host.numpy()
            host[: len(p)] = p
            host[len(p):] = np.nan
        if self.provider is not None:
            from .query import query_min_distances, voxelize_pointcloud

            obs = voxelize_pointcloud(self.p_host.to("cuda", non_blocking=True), self.grid)
            return query_min_distances(self.field, obs, return_argmin=True)
        if self._graph is not None:
            self._graph.replay()
        else:
            self._run()
        t.cuda.current_stream().synchronize()
        return tuple(self.out_host[k].numpy().copy() for k in ("d", "link", "voxel"))


class ShardedCloudPipeline(_CycleResults):
    """CheckerPipeline for one rank of a multi-GPU throughput sweep whose cloud
    is shared: each rank uploads only ITS slice of the points (and of the
    waypoints), voxelizes the slice, and the ranks all-gather their partial
    occupancy bitmaps (ceil(V/32) words each) and dropped counters over
    NVLink; ``lsdf_occupancy_merge`` ORs them into the full occupancy.  Per
    cycle a rank moves 1/world of the cloud over PCIe instead of all of it;
    the exchange is 16 KB per rank at 50^3.  Results are those of one rank
    voxelizing the whole cloud (tests: ``test_sharded_cloud_pipeline``).

    Producers fill ``inputs()`` (pinned configs of this rank's waypoints,
    pinned points of this rank's slice, NaN-padded), then ``submit()``;
    ``result(ticket)`` returns this rank's (d, link, voxel).
    """

    def __init__(self, robot, sdfs, grid, window, n_configs: int, n_points_local: int, points_dtype=np.float32,
                 depth: int = 2, group=None, **kw):
        import torch.distributed as dist

        t = N.torch()
        self.group = group
        self.world = dist.get_world_size(group)
        self.grid = grid
        n_words = (grid.n_voxels + 31) // 32
        self._bits = slice(256 // 4, 256 // 4 + n_words)  # int32 view of the occupancy workspace
        self.slots = []
        for _ in range(depth):
            chk = DistanceChecker(robot, sdfs, grid, window, **kw).prepare(
                n_configs, n_points_local, points_dtype, use_graph=False, zero_copy=False)
            pin = dict(pin_memory=True)
            host_out = (t.zeros((n_configs,), dtype=t.float32, **pin), t.zeros((n_configs,), dtype=t.int32, **pin),
                        t.zeros((n_configs,), dtype=t.int32, **pin), t.zeros((4,), dtype=t.int32, **pin))
            part = occupancy_workspace(grid)
            gather = N.empty((self.world, n_words), t.int32)
            dropped = N.empty((self.world,), t.int32)
            ev = {k: t.cuda.Event() for k in ("h2d", "compute", "d2h")}
            self.slots.append({"chk": chk, "out": host_out, "part": part, "gather": gather, "dropped": dropped,
                               "ev": ev, "busy": False, "ticket": -1})
        self.copy = t.cuda.Stream()
        self.compute = t.cuda.Stream()
        self.d2h = t.cuda.Stream()
        self._next = 0
        self._done = {}

    @property
    def depth(self) -> int:
        return len(self.slots)

    def _slot(self, ticket):
        return self.slots[ticket % len(self.slots)]

    def inputs(self):
        s = self._slot(self._next)
        if s["busy"]:
            self._drain(s)
        return s["chk"].host_inputs()

    def _all_gather(self, out, inp):
        import torch.distributed as dist

        try:
            dist.all_gather_into_tensor(out, inp, group=self.group)
        except (RuntimeError, NotImplementedError):  # backends without the flat form (gloo)
            dist.all_gather(list(out.unbind(0)), inp, group=self.group)

    def submit(self) -> int:
        t = N.torch()
        ticket = self._next
        s = self._slot(ticket)
        if s["busy"]:
            self._drain(s)
        chk, ev = s["chk"], s["ev"]
        C_, P, pdt = chk._shape
        with t.cuda.stream(self.copy):
            self.copy.wait_event(ev["compute"])
            chk.q_dev.copy_(chk.q_host, non_blocking=True)
            chk.p_dev.copy_(chk.p_host, non_blocking=True)
            ev["h2d"].record(self.copy)
        with t.cuda.stream(self.compute):
            self.compute.wait_event(ev["h2d"])
            self.compute.wait_event(ev["d2h"])
            cs = self.compute.cuda_stream
            N.call(chk._fk_entry, chk._chain, chk.robot.n_links, len(chk.sdfs), N.ptr(chk.q_dev), C_,
                   chk.robot.dof, N.ptr(chk.limits), chk._env, chk._W, None, None, N.ptr(chk.R_geo),
                   N.ptr(chk.dt_geo), N.ptr(chk.anchor_geo), N.ptr(chk.flags), cs)
            part = s["part"].view(t.int32)
            N.call("lsdf_voxelize_bitmap", N.ptr(chk.p_dev), int(pdt == np.float32), P, chk._env, s["part"], cs)
            self._all_gather(s["gather"], part[self._bits])
            self._all_gather(s["dropped"], part[1:2])  # counters[1]: dropped points of the slice
            N.call("lsdf_occupancy_merge", s["gather"], self.world, s["dropped"], 1, chk._env, N.ptr(chk.ws), cs)
            tr = chk.traj
            N.call("lsdf_query_direct", N.ptr(chk.R_geo), N.ptr(chk.dt_geo), N.ptr(chk.anchor_geo), C_, tr.n_links,
                   tr._table, ctypes.byref(chk._wstruct), chk._env, N.ptr(chk.ws), chk._qflags, chk.d_far_global,
                   N.ptr(chk.qws), N.ptr(chk.d_dev), N.ptr(chk.link_dev), N.ptr(chk.voxel_dev), None, cs)
            ev["compute"].record(self.compute)
        d, link, voxel, flags = s["out"]
        with t.cuda.stream(self.d2h):
            self.d2h.wait_event(ev["compute"])
            d.copy_(chk.d_dev, non_blocking=True)
            link.copy_(chk.link_dev, non_blocking=True)
            voxel.copy_(chk.voxel_dev, non_blocking=True)
            flags.copy_(chk.flags[:4], non_blocking=True)
            ev["d2h"].record(self.d2h)
        s["busy"], s["ticket"] = True, ticket
        self._next += 1
        return ticket
