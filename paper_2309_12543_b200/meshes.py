"""Collision geometry and the link-SDF precompute (stage 2a).

Host-side mirror of the reference ``meshes.py``: primitive/mesh types, mesh
construction and file loaders are host plumbing (meshes.py:25-141, 378-534);
``primitive_sdf``, ``exact_point_distance`` and ``build_link_sdf`` run the
CUDA kernels in ``csrc/lsdf_build.cu`` (fp64, the reference's operation
order, f32 store).
"""

from __future__ import annotations

import ctypes
import logging
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import NonWatertightError, ValidationError

log = logging.getLogger(__name__)


@dataclass(frozen=True, eq=False)
class Sphere:
    radius: float
    center: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=np.float64))


@dataclass(frozen=True, eq=False)
class Capsule:
    """Segment of +-half_length along ``axis`` through the origin, inflated by radius."""

    radius: float
    half_length: float
    axis: np.ndarray = field(default_factory=lambda: np.float64([0.0, 0.0, 1.0]))

    def __post_init__(self):
        axis = np.asarray(self.axis, dtype=np.float64)
        n = np.linalg.norm(axis)
        if n == 0:
            raise ValidationError("capsule axis must be nonzero")
        object.__setattr__(self, "axis", axis / n)


@dataclass(frozen=True, eq=False)
class Box:
    half_extents: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "half_extents", np.asarray(self.half_extents, dtype=np.float64))


Primitive = Sphere | Capsule | Box


def _primitive_params(shape) -> tuple[int, ctypes.Array]:
    p = np.zeros(8)
    if isinstance(shape, Sphere):
        p[0] = shape.radius
        p[1:4] = shape.center
        return 0, N.f64s(p, 8)
    if isinstance(shape, Capsule):
        p[0], p[1] = shape.radius, shape.half_length
        p[2:5] = shape.axis
        return 1, N.f64s(p, 8)
    if isinstance(shape, Box):
        p[0:3] = shape.half_extents
        return 2, N.f64s(p, 8)
    raise ValidationError(f"unknown primitive {type(shape).__name__}")


def primitive_sdf(shape, points) -> np.ndarray:
    """Analytic signed distance, negative inside (meshes.py:64-82), on the GPU."""
    kind, prm = _primitive_params(shape)
    pts = np.asarray(points, dtype=np.float64)
    scalar = pts.ndim == 1
    flat = np.ascontiguousarray(pts.reshape(-1, 3))
    t = N.torch()
    d_pts = N.to_device(flat, t.float64)
    out = N.empty((len(flat),), t.float64)
    N.call("lsdf_primitive_points", kind, prm, N.ptr(d_pts), len(flat), N.ptr(out), N.stream())
    d = out.cpu().numpy()
    return d[0] if scalar else d.reshape(pts.shape[:-1])


def _morton_order(points: np.ndarray) -> np.ndarray:
    """Permutation sorting points along a 3-D Z-order curve (10 bits per axis)."""
    p = np.asarray(points, dtype=np.float64)
    lo, hi = p.min(axis=0), p.max(axis=0)
    q = np.clip(((p - lo) / np.maximum(hi - lo, 1e-300) * 1023.0).astype(np.int64), 0, 1023)

    def spread(v):
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        return (v | (v << 2)) & 0x09249249

    code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    return np.argsort(code, kind="stable")


class TriangleMesh:
    """Triangle soup with load-time removal of degenerate faces (meshes.py:85-141)."""

    def __init__(self, vertices, triangles):
        vertices = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        triangles = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
        if triangles.size and (triangles.min() < 0 or triangles.max() >= len(vertices)):
            raise ValidationError("triangle indices out of range")
        a, b, c = vertices[triangles[:, 0]], vertices[triangles[:, 1]], vertices[triangles[:, 2]]
        keep = np.linalg.norm(np.cross(b - a, c - a), axis=-1) > 1e-14
        dropped = int((~keep).sum())
        if dropped:
            log.warning("dropped %d degenerate triangle(s)", dropped)
            triangles = triangles[keep]
        if len(triangles) == 0:
            raise ValidationError("mesh has no non-degenerate triangles")
        self.vertices = vertices
        self.triangles = triangles
        self.vertices.flags.writeable = False
        self.triangles.flags.writeable = False
        self._watertight = None
        self._dev = None

    @property
    def is_watertight(self) -> bool:
        """Every undirected edge is shared by exactly two triangles."""
        if self._watertight is None:
            t = self.triangles
            edges = np.sort(np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
            _, counts = np.unique(edges, axis=0, return_counts=True)
            self._watertight = bool(np.all(counts == 2))
        return self._watertight

    def triangle_corners(self):
        v, t = self.vertices, self.triangles
        return v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]

    def device_corners(self):
        """(T, 9) fp64 corner table on the GPU (a, b, c per row), cached.

        Rows are in Morton order of the triangle centroids, so each 128-row
        tile of the build kernel covers a compact patch of the surface and its
        box culls well; every per-cell result (a min and a crossing parity)
        is independent of the triangle order.
        """
        if self._dev is None:
            a, b, c = self.triangle_corners()
            table = np.concatenate([a, b, c], axis=1)
            table = table[_morton_order((a + b + c) / 3.0)]
            self._dev = N.to_device(np.ascontiguousarray(table), N.torch().float64)
        return self._dev

    def sample_surface(self, n: int, rng: np.random.Generator) -> np.ndarray:
        a, b, c = self.triangle_corners()
        areas = 0.5 * np.linalg.norm(np.cross(b - a, c - a), axis=-1)
        which = rng.choice(len(areas), size=n, p=areas / areas.sum())
        u = rng.random(n)
        v = rng.random(n)
        flip = u + v > 1.0
        u[flip] = 1.0 - u[flip]
        v[flip] = 1.0 - v[flip]
        return a[which] + u[:, None] * (b[which] - a[which]) + v[:, None] * (c[which] - a[which])


def exact_point_distance(mesh: TriangleMesh, points, signed: bool = True) -> np.ndarray:
    """Exact point-to-surface distance, ray-parity sign (meshes.py:308-329), on the GPU."""
    if signed and not mesh.is_watertight:
        raise NonWatertightError("signed distance requested on an open mesh; pass signed=False")
    pts = np.asarray(points, dtype=np.float64)
    scalar = pts.ndim == 1
    flat = np.ascontiguousarray(pts.reshape(-1, 3))
    t = N.torch()
    d_pts = N.to_device(flat, t.float64)
    out = N.empty((len(flat),), t.float64)
    N.call("lsdf_mesh_points", N.ptr(mesh.device_corners()), len(mesh.triangles), int(signed),
           N.ptr(d_pts), len(flat), N.ptr(out), N.stream())
    d = out.cpu().numpy()
    return float(d[0]) if scalar else d.reshape(pts.shape[:-1])


def build_link_sdf(geometry, extent, resolution, link_id: int = 0):
    """Bake a link's geometry into a dense exact SDF grid (meshes.py:332-371).

    Runs entirely on the GPU; the returned LinkSdf keeps its values resident
    in device memory (host view materialised on first ``.values`` access).
    """
    from .grids import LinkSdf

    ext = np.broadcast_to(np.asarray(extent, dtype=np.float64), (3,)).copy()
    res = np.broadcast_to(np.asarray(resolution, dtype=np.float64), (3,)).copy()
    dims = np.rint(2.0 * ext / res).astype(np.int64)
    t = N.torch()
    out = N.empty((int(np.prod(dims)),), t.float32)
    if isinstance(geometry, TriangleMesh):
        signed = geometry.is_watertight
        if not signed:
            log.warning("link %d: mesh is not watertight, storing unsigned distances", link_id)
        N.call("lsdf_build_mesh", N.ptr(geometry.device_corners()), len(geometry.triangles),
               int(signed), N.f64s(ext, 3), N.f64s(res, 3), N.i32x3(dims), N.ptr(out), N.stream())
    else:
        kind, prm = _primitive_params(geometry)
        N.call("lsdf_build_primitive", kind, prm, N.f64s(ext, 3), N.f64s(res, 3), N.i32x3(dims),
               N.ptr(out), N.stream())
    return LinkSdf(extent=ext, resolution=res, values=out, link_id=link_id)


# --------------------------------------------------------------------------- constructors / IO


def make_box_mesh(half_extents) -> TriangleMesh:
    """Axis-aligned box, 12 outward-facing triangles."""
    h = np.asarray(half_extents, dtype=np.float64)
    corners = np.array([[x, y, z] for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)],
                       dtype=np.float64) * h
    quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    tris = [t for q in quads for t in ((q[0], q[1], q[2]), (q[0], q[2], q[3]))]
    return TriangleMesh(corners, np.int64(tris))


def make_icosphere(radius: float, subdivisions: int = 1) -> TriangleMesh:
    """Subdivided icosahedron projected to the sphere (80 faces at 1 subdivision)."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    base = np.float64([[-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0],
                       [0, -1, phi], [0, 1, phi], [0, -1, -phi], [0, 1, -phi],
                       [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1]])
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    verts = [v / np.linalg.norm(v) for v in base]
    for _ in range(subdivisions):
        mids: dict = {}

        def mid(i, j):
            key = (min(i, j), max(i, j))
            if key not in mids:
                m = verts[i] + verts[j]
                verts.append(m / np.linalg.norm(m))
                mids[key] = len(verts) - 1
            return mids[key]

        nxt = []
        for i, j, k in faces:
            ij, jk, ki = mid(i, j), mid(j, k), mid(k, i)
            nxt += [(i, ij, ki), (j, jk, ij), (k, ki, jk), (ij, jk, ki)]
        faces = nxt
    return TriangleMesh(np.float64(verts) * radius, np.int64(faces))


def primitive_surface_points(shape, n: int, rng: np.random.Generator):
    """Random points on a primitive's surface (coverage validation)."""
    if isinstance(shape, Sphere):
        d = rng.normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=-1, keepdims=True)
        return shape.center + shape.radius * d
    if isinstance(shape, Capsule):
        d = rng.normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=-1, keepdims=True)
        t = rng.uniform(-shape.half_length, shape.half_length, size=n)
        axial = d @ shape.axis
        radial = d - axial[:, None] * shape.axis
        on_cap = rng.random(n) < (2 * shape.radius / (2 * shape.radius + 2 * shape.half_length))
        return np.where(
            on_cap[:, None],
            np.sign(axial)[:, None] * shape.half_length * shape.axis + shape.radius * d,
            t[:, None] * shape.axis
            + shape.radius * radial / np.maximum(np.linalg.norm(radial, axis=-1, keepdims=True), 1e-12))
    if isinstance(shape, Box):
        return make_box_mesh(shape.half_extents).sample_surface(n, rng)
    raise ValidationError(f"unknown primitive {type(shape).__name__}")


def load_stl(path) -> TriangleMesh:
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:5] == b"solid" and b"facet" in data[:2048]:
        coords = [[float(x) for x in ln.split()[1:]] for ln in data.decode("ascii", "replace").splitlines()
                  if len(ln.split()) == 4 and ln.split()[0] == "vertex"]
        return _from_soup(np.float64(coords).reshape(-1, 3, 3))
    if len(data) < 84:
        raise ValidationError(f"{path}: truncated STL")
    (count,) = struct.unpack_from("<I", data, 80)
    if len(data) < 84 + 50 * count:
        raise ValidationError(f"{path}: STL facet data truncated")
    raw = np.frombuffer(data, dtype=np.uint8, count=50 * count, offset=84).reshape(count, 50)
    return _from_soup(raw[:, 12:48].copy().view("<f4").reshape(count, 3, 3).astype(np.float64))


def load_obj(path) -> TriangleMesh:
    vertices, faces = [], []
    with open(path) as fh:
        for line in fh:
            parts = line.split()
            if not parts:
                continue
            if parts[0] == "v":
                vertices.append([float(x) for x in parts[1:4]])
            elif parts[0] == "f":
                idx = [int(p.split("/")[0]) - 1 for p in parts[1:]]
                faces += [(idx[0], idx[i], idx[i + 1]) for i in range(1, len(idx) - 1)]
    return TriangleMesh(np.float64(vertices), np.int64(faces))


def load_mesh(path) -> TriangleMesh:
    p = str(path).lower()
    if p.endswith(".stl"):
        return load_stl(path)
    if p.endswith(".obj"):
        return load_obj(path)
    raise ValidationError(f"unsupported mesh format: {path}")


def _from_soup(tris: np.ndarray) -> TriangleMesh:
    verts, inverse = np.unique(tris.reshape(-1, 3), axis=0, return_inverse=True)
    return TriangleMesh(verts, inverse.reshape(-1, 3))
