"""Alignment and resampling of link SDFs onto the environment grid.

Host-side mirror of the reference ``placement.py`` (placement.py:29-313).
The window tables (canonical points, ball mask) are per-(extent, grid)
constants built on the host with the reference's own numpy expressions and
uploaded once (``WindowGeometry.device_tables``): the normalized offsets per
axis, the keep-mask as a bit table, and per window column the z-interval of
kept cells that the fused query kernel iterates.  ``compute_alignment``,
``grid_transform_exact`` and ``place_links_batch`` run CUDA kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterator, Protocol, Sequence

import numpy as np

from . import _native as N
from .errors import NoOverlapError, ValidationError
from .grids import EnvGrid, LinkSdf, SdfSampleField

_ISOTROPY_RTOL = 1e-9


def window_dims(extent_r, grid: EnvGrid) -> np.ndarray:
    """Window width per axis, 2*e_r/r_e, which must be an even integer (placement.py:29-44)."""
    extent_r = np.broadcast_to(np.asarray(extent_r, dtype=np.float64), (3,))
    ratio = 2.0 * extent_r / grid.resolution
    dims = np.rint(ratio)
    if np.any(np.abs(ratio - dims) > 1e-6 * np.maximum(ratio, 1.0)):
        raise ValidationError(f"link extent {extent_r} is not an integer multiple of the "
                              f"environment resolution {grid.resolution}")
    dims = dims.astype(np.int64)
    if np.any(dims % 2 != 0):
        raise ValidationError(f"window width must be even per axis, got {dims}")
    if np.any(dims < 2):
        raise ValidationError(f"window width must be at least 2, got {dims}")
    return dims


@dataclass(frozen=True, eq=False)
class AlignmentResult:
    """Window anchor + sub-voxel residual: voxel_center(anchor + W/2) + delta_t == T."""

    anchor: np.ndarray
    delta_t: np.ndarray


def _align_device(T_dev, grid: EnvGrid, W):
    t = N.torch()
    n = int(T_dev.shape[0])
    anchor = N.empty((n, 3), t.int32)
    dt = N.empty((n, 3), t.float64)
    flags = N.zeros((4,), t.int32)
    N.call("lsdf_align", N.ptr(T_dev), n, ctypes.byref(grid.c_struct()), N.i32x3(W), N.ptr(anchor),
           N.ptr(dt), N.ptr(flags), N.stream())
    return anchor, dt, flags


def compute_alignment(translation, grid: EnvGrid, extent_r) -> AlignmentResult:
    """Split positions into voxel anchors and residuals (placement.py:60-99), on the GPU.

    Raises NoOverlapError when a window misses the grid entirely.
    """
    w = window_dims(extent_r, grid)
    tr = np.asarray(translation, dtype=np.float64)
    scalar = tr.ndim == 1
    pos = np.ascontiguousarray(tr.reshape(-1, 3))
    anchor_d, dt_d, flags = _align_device(N.to_device(pos, N.torch().float64), grid, w)
    anchor = anchor_d.cpu().numpy().astype(np.int64)
    delta = dt_d.cpu().numpy()
    bad = int(flags[1].item())
    if bad:
        outside = np.any((anchor >= grid.dims) | (anchor + w <= 0), axis=-1)
        raise NoOverlapError(f"{bad} window(s) miss the grid entirely, e.g. at {pos[np.argmax(outside)].tolist()}")
    if scalar:
        return AlignmentResult(anchor=anchor[0], delta_t=delta[0])
    return AlignmentResult(anchor=anchor.reshape(tr.shape[:-1] + (3,)), delta_t=delta.reshape(tr.shape))


def _iso_extent(extent_r) -> float:
    extent_r = np.broadcast_to(np.asarray(extent_r, dtype=np.float64), (3,))
    if np.any(np.abs(extent_r - extent_r[0]) > _ISOTROPY_RTOL * extent_r[0]):
        raise ValidationError(f"placement requires an isotropic link extent, got {extent_r}")
    return float(extent_r[0])


def _axis_offsets(extent_r, grid: EnvGrid, normalized: bool):
    e_r = _iso_extent(extent_r)
    w = window_dims(extent_r, grid)
    if normalized:
        return [(np.arange(w[a]) - w[a] // 2) * grid.resolution[a] / e_r for a in range(3)]
    return [(np.arange(w[a]) - w[a] // 2) * grid.resolution[a] for a in range(3)]


def canonical_points(extent_r, grid: EnvGrid) -> np.ndarray:
    """Normalized window cell centres, x-fastest (placement.py:112-125)."""
    ax = _axis_offsets(extent_r, grid, True)
    zz, yy, xx = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return np.stack([xx, yy, zz], axis=-1).reshape(-1, 3)


def sphere_mask(extent_r, grid: EnvGrid) -> np.ndarray:
    """Keep-mask (Wx, Wy, Wz): centre strictly within e_r of the window centre (placement.py:128-145)."""
    e_r = _iso_extent(extent_r)
    ax = _axis_offsets(extent_r, grid, False)
    xx, yy, zz = np.meshgrid(ax[0], ax[1], ax[2], indexing="ij")
    return xx * xx + yy * yy + zz * zz < e_r * e_r * (1.0 - 1e-12)


def grid_transform_exact(rotations, delta_t, extent_r, points):
    """G = P R + dt_inv with dt_inv = -(dt/e_r) R (placement.py:148-169), on the GPU."""
    e_r = _iso_extent(extent_r)
    r = np.asarray(rotations, dtype=np.float64)
    single = r.ndim == 2
    r = np.ascontiguousarray(r.reshape(-1, 3, 3))
    dt = np.ascontiguousarray(np.asarray(delta_t, dtype=np.float64).reshape(-1, 3))
    P = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    t = N.torch()
    G = N.empty((len(r), len(P), 3), t.float64)
    N.call("lsdf_grid_transform_exact", N.to_device(r, t.float64), N.to_device(dt, t.float64),
           len(r), N.to_device(P, t.float64), len(P), e_r, N.ptr(G), N.stream())
    g = G.cpu().numpy()
    return g[0] if single else g


class WindowGeometry:
    """Per-(extent, grid) placement constants shared by all links and poses (placement.py:172-210)."""

    def __init__(self, grid, extent, dims, points, mask, masked_points):
        self.grid = grid
        self.extent = extent
        self.dims = dims
        self.points = points
        self.mask = mask
        self.masked_points = masked_points
        self._tables = None

    @classmethod
    def build(cls, extent_r, grid: EnvGrid) -> "WindowGeometry":
        e_r = _iso_extent(extent_r)
        dims = window_dims(extent_r, grid)
        points = canonical_points(extent_r, grid)
        mask = sphere_mask(extent_r, grid)
        return cls(grid=grid, extent=e_r, dims=dims, points=points, mask=mask,
                   masked_points=points[mask.ravel(order="F")])

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.dims))

    @property
    def n_masked(self) -> int:
        return len(self.masked_points)

    def matches_link(self, sdf: LinkSdf) -> bool:
        return bool(np.all(np.abs(sdf.extent - self.extent) <= 1e-9 * self.extent))

    def host_tables(self) -> dict:
        """The ``lsdf_window`` tables as host arrays (what ``device_tables`` uploads).

        P (3, Wmax) f64 normalized offsets; zrange (W1*W0, 2) i16 or None when a
        column's kept cells are not one z interval; mask_bits u32; shell_cells
        u32 / shell_radius f32 (kept cells by distance from the window centre,
        radius rounded down; padded to a multiple of 32 with the last cell); kept_cells i32 (x-fastest order).
        """
        W = [int(d) for d in self.dims]
        if max(W) > 256:
            raise ValidationError(f"window width {W} exceeds the supported 256 cells")
        Wmax = max(W)
        P = np.zeros((3, Wmax))
        for a, off in enumerate(_axis_offsets(self.extent, self.grid, True)):
            P[a, : W[a]] = off
        mask_f = self.mask.ravel(order="F")
        bits = np.zeros(((len(mask_f) + 31) // 32) * 32, dtype=np.uint8)
        bits[: len(mask_f)] = mask_f
        words = np.packbits(bits.reshape(-1, 32)[:, ::-1], axis=1).view(">u4").ravel().astype(np.uint32)
        # per (mx, my) column: the kept z cells form one interval [lo, hi)
        zr = np.zeros((W[1], W[0], 2), dtype=np.int16)
        interval = True
        for my in range(W[1]):
            for mx in range(W[0]):
                zs = np.nonzero(self.mask[mx, my, :])[0]
                if len(zs):
                    zr[my, mx] = (zs[0], zs[-1] + 1)
                    interval &= bool(len(zs) == zs[-1] + 1 - zs[0])
        # kept cells sorted by distance from the window centre (shell order)
        off = _axis_offsets(self.extent, self.grid, False)
        mxs, mys, mzs = np.nonzero(self.mask)
        dist = np.sqrt(off[0][mxs] ** 2 + off[1][mys] ** 2 + off[2][mzs] ** 2)
        order = np.argsort(dist, kind="stable")
        packed = (mxs | (mys << 8) | (mzs << 16)).astype(np.uint32)[order]
        radius = np.nextafter(dist[order].astype(np.float32), np.float32(-np.inf))  # rounded down
        radius = np.minimum(radius, dist[order]).astype(np.float32)
        # padded to whole 32-cell chunks with copies of the last cell: the scan
        # needs no per-lane bound check, and a repeated cell changes no minimum
        pad = -len(packed) % 32
        if pad and len(packed):
            packed = np.concatenate([packed, np.repeat(packed[-1:], pad)])
            radius = np.concatenate([radius, np.repeat(radius[-1:], pad)])
        return {"W": W, "Wmax": Wmax, "n_masked": self.n_masked, "e_r": float(self.extent), "P": P,
                "zrange": zr.reshape(-1, 2) if interval else None, "mask_bits": words,
                "shell_cells": packed, "shell_radius": radius,
                "kept_cells": np.nonzero(mask_f)[0].astype(np.int32)}

    def device_tables(self):
        """Upload (once) the host tables; returns (``lsdf_window`` struct, tensors)."""
        if self._tables is not None:
            return self._tables
        t = N.torch()
        h = self.host_tables()
        dev = {
            "P": N.to_device(h["P"], t.float64),
            "mask_bits": N.to_device(h["mask_bits"].view(np.int32), t.int32),
            "zrange": N.to_device(h["zrange"], t.int16) if h["zrange"] is not None else None,
            "kept_cells": N.to_device(h["kept_cells"], t.int32),
            "shell_cells": N.to_device(h["shell_cells"].view(np.int32), t.int32),
            "shell_radius": N.to_device(h["shell_radius"], t.float32),
        }
        s = N.WindowT()
        s.W[:] = h["W"]
        s.n_masked = h["n_masked"]
        s.e_r = h["e_r"]
        s.P_dev = N.ptr(dev["P"])
        s.Wmax = h["Wmax"]
        s.zrange_dev = N.ptr(dev["zrange"])
        s.mask_bits_dev = N.ptr(dev["mask_bits"])
        s.shell_cells_dev = N.ptr(dev["shell_cells"])
        s.shell_radius_dev = N.ptr(dev["shell_radius"])
        self._tables = (s, dev)
        return self._tables


class TransformProvider(Protocol):
    """Maps poses to normalized link-frame sample coordinates of the kept window cells."""

    window: WindowGeometry

    def transform(self, rotations: np.ndarray, delta_t: np.ndarray) -> np.ndarray:
        """(B, 3, 3), (B, 3) -> (B, n_masked, 3)."""
        ...


class ExactTransformProvider:
    """Deterministic P R transform; the fused kernels evaluate it in place."""

    def __init__(self, window: WindowGeometry):
        self.window = window

    def transform(self, rotations, delta_t):
        return grid_transform_exact(rotations, delta_t, self.window.extent, self.window.masked_points)


def link_grid_table(sdfs: Sequence[LinkSdf], packed: bool = False, packed_ptrs=None):
    table = (N.LinkGridT * len(sdfs))()
    for i, s in enumerate(sdfs):
        table[i] = s.c_struct(packed)
        if packed_ptrs is not None:
            table[i].packed_dev = packed_ptrs[i]
    return table


def packed_arena(sdfs: Sequence[LinkSdf]):
    """One contiguous device copy of the links' packed-corner grids and each link's address in it.

    Contiguity lets the query mark every grid it reads persisting in L2 with
    a single access-policy window (lsdf_l2_reserve).
    """
    t = N.torch()
    parts = [s.packed_values() for s in sdfs]
    arena = t.cat(parts) if len(parts) > 1 else parts[0].clone()
    ptrs, off = [], 0
    for part in parts:
        ptrs.append(N.ptr(arena) + off * 4)
        off += int(part.numel())
    return arena, ptrs


def _check_links(sdfs, window: WindowGeometry):
    for sdf in sdfs:
        if not window.matches_link(sdf):
            raise ValidationError(f"link {sdf.link_id}: extent {sdf.extent} does not match "
                                  f"provider window extent {window.extent}")


def place_windows_device(sdfs, R_dev, dt_dev, window: WindowGeometry, provider=None):
    """Every (c, l) window as a (C, L, W^3) f32 CUDA tensor (x-fastest cells)."""
    t = N.torch()
    C_, L = int(R_dev.shape[0]), int(R_dev.shape[1])
    out = N.empty((C_, L, window.n_cells), t.float32)
    if provider is None or isinstance(provider, ExactTransformProvider):
        ws, _ = window.device_tables()
        N.call("lsdf_place_windows", N.ptr(R_dev), N.ptr(dt_dev), C_, L, link_grid_table(sdfs, packed=True),
               ctypes.byref(ws), N.ptr(out), N.stream())
        return out
    ws, dev = window.device_tables()
    from .approx import NeuralTransformProvider

    if isinstance(provider, NeuralTransformProvider):
        # the neural provider stays on the device: TinyMlp on the tensor cores
        # (or the CUDA-core sgemm replica), then the provider-coordinate sampler
        if provider.fused:
            m = provider.model
            w1, b1, _, b2 = m.device_weights()
            N.call("lsdf_mlp_place", w1, b1, m.packed_w2_cells(), b2, m.hidden, m.n_points, dev["kept_cells"],
                   N.ptr(R_dev), N.ptr(dt_dev), C_, L, link_grid_table(sdfs, packed=True), ctypes.byref(ws), out,
                   N.stream())
            return out
        R_flat = R_dev.reshape(C_ * L, 9)
        y = provider.model.predict_device(R_flat, use_tensor_cores=provider.use_tensor_cores)
        N.call("lsdf_place_windows_g", y, int(y.stride(0)), dev["kept_cells"], window.n_masked, N.ptr(R_dev),
               N.ptr(dt_dev), C_, L,
               link_grid_table(sdfs, packed=True), ctypes.byref(ws), out, N.stream())
        return out
    # generic provider: its coordinates (host), our sampler (placement.py:300-313)
    mask_f = t.from_numpy(window.mask.ravel(order="F")).to(out.device)
    for li, sdf in enumerate(sdfs):
        G = provider.transform(R_dev[:, li].cpu().numpy(), dt_dev[:, li].cpu().numpy())
        G = N.to_device(G, t.float64).reshape(-1, 3)
        samples = N.empty((G.shape[0],), t.float32)
        g = sdf.c_struct()
        N.call("lsdf_trilinear", ctypes.byref(g), N.ptr(G), int(G.shape[0]), float(window.extent),
               N.ptr(samples), N.stream())
        blk = t.full((C_, window.n_cells), float(np.float32(sdf.d_far)), dtype=t.float32, device=out.device)
        blk[:, mask_f] = samples.reshape(C_, -1)
        out[:, li] = blk
    return out


def place_link(sdf: LinkSdf, rotation, translation, grid: EnvGrid, provider) -> SdfSampleField:
    """Resample one link SDF onto its environment-aligned window (placement.py:235-264)."""
    window = provider.window
    if not window.matches_link(sdf):
        raise ValidationError(f"provider window extent {window.extent} does not match link extent {sdf.extent}")
    from .robot import LinkPoseBatch

    poses = LinkPoseBatch(rotations=np.asarray(rotation, dtype=np.float64).reshape(1, 1, 3, 3),
                          translations=np.asarray(translation, dtype=np.float64).reshape(1, 1, 3))
    (_, _, field), = list(place_links_batch([sdf], poses, grid, provider))
    return field


def place_links_batch(sdfs: Sequence[LinkSdf], poses, grid: EnvGrid, provider,
                      chunk: int = 8) -> Iterator[tuple[int, int, SdfSampleField]]:
    """Resample every (configuration, link) pair (placement.py:267-313).

    All windows are computed in one GPU pass; the generator then yields
    (config_index, link_index, field) grouped by link, like the reference.
    ``chunk`` is accepted for signature compatibility (the GPU needs no
    host-side chunking).
    """
    window = provider.window
    C_, L = poses.n_configs, poses.n_links
    if len(sdfs) != L:
        raise ValidationError(f"{len(sdfs)} SDFs for {L} links")
    _check_links(sdfs, window)
    t = N.torch()
    R = N.to_device(np.ascontiguousarray(poses.rotations, dtype=np.float64), t.float64)
    T = N.to_device(np.ascontiguousarray(np.asarray(poses.translations, dtype=np.float64).reshape(-1, 3)),
                    t.float64)
    anchor_d, dt_d, flags = _align_device(T, grid, window.dims)
    if int(flags[1].item()):
        anchor = anchor_d.cpu().numpy()
        outside = np.any((anchor >= grid.dims) | (anchor + window.dims <= 0), axis=-1)
        raise NoOverlapError(f"{int(outside.sum())} window(s) miss the grid entirely, "
                             f"e.g. at {T[int(np.argmax(outside))].cpu().numpy().tolist()}")
    vals = place_windows_device(sdfs, R, dt_d.reshape(C_, L, 3), window, provider).cpu().numpy()
    anchors = anchor_d.cpu().numpy().astype(np.int64).reshape(C_, L, 3)
    shape = tuple(int(d) for d in window.dims)
    for li in range(L):
        d_far = sdfs[li].d_far
        for c in range(C_):
            yield c, li, SdfSampleField(values=vals[c, li].reshape(shape, order="F"),
                                        anchor=anchors[c, li], d_far=d_far)
