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


def _vec(v) -> np.ndarray:
    return np.asarray(v, dtype=np.float64)


@dataclass(frozen=True, eq=False)
class Sphere:
    """Ball of ``radius`` about ``center`` (link frame)."""

    radius: float
    center: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        object.__setattr__(self, "center", _vec(self.center))


@dataclass(frozen=True, eq=False)
class Capsule:
    """Segment of +-half_length along ``axis`` through the origin, inflated by radius."""

    radius: float
    half_length: float
    axis: np.ndarray = field(default_factory=lambda: np.float64([0.0, 0.0, 1.0]))

    def __post_init__(self):
        direction = _vec(self.axis)
        length = np.linalg.norm(direction)
        if not length:
            raise ValidationError("capsule axis must be nonzero")
        object.__setattr__(self, "axis", direction / length)


@dataclass(frozen=True, eq=False)
class Box:
    """Axis-aligned box of the given half extents about the link origin."""

    half_extents: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "half_extents", _vec(self.half_extents))


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
    """Indexed triangle soup (meshes.py:85-141); zero-area faces are dropped
    (with a warning) when the mesh is built."""

    def __init__(self, vertices, triangles):
        v = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        f = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
        if f.size and not (0 <= f.min() and f.max() < len(v)):
            raise ValidationError("triangle indices out of range")
        corners = v[f]  # (T, 3 corners, 3)
        twice_area = np.linalg.norm(np.cross(corners[:, 1] - corners[:, 0], corners[:, 2] - corners[:, 0]), axis=-1)
        degenerate = twice_area <= 1e-14
        if degenerate.any():
            log.warning("dropped %d degenerate triangle(s)", int(degenerate.sum()))
            f = f[~degenerate]
        if not len(f):
            raise ValidationError("mesh has no non-degenerate triangles")
        v.flags.writeable = False
        f.flags.writeable = False
        self.vertices, self.triangles = v, f
        self._watertight = None
        self._dev = None

    @property
    def is_watertight(self) -> bool:
        """Closed 2-manifold test: each undirected edge belongs to exactly two faces."""
        if self._watertight is None:
            f = self.triangles
            ends = np.sort(np.stack([f, np.roll(f, -1, axis=1)], axis=-1).reshape(-1, 2), axis=1)
            key = ends[:, 0] * (int(f.max()) + 1) + ends[:, 1]
            _, uses = np.unique(key, return_counts=True)
            self._watertight = bool((uses == 2).all())
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
        """n area-weighted surface points; draws from ``rng`` in the reference's
        order (face choice, then u, then v; folded barycentrics)."""
        a, b, c = self.triangle_corners()
        weight = np.linalg.norm(np.cross(b - a, c - a), axis=-1) * 0.5
        face = rng.choice(len(weight), size=n, p=weight / weight.sum())
        uv = np.stack([rng.random(n), rng.random(n)], axis=1)
        outside = uv.sum(axis=1) > 1.0
        uv[outside] = 1.0 - uv[outside]
        return a[face] + uv[:, :1] * (b[face] - a[face]) + uv[:, 1:] * (c[face] - a[face])


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


def _unit_normals(rng: np.random.Generator, n: int) -> np.ndarray:
    d = rng.normal(size=(n, 3))
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def primitive_surface_points(shape, n: int, rng: np.random.Generator):
    """Random points on a primitive's surface (sphere-model validation); the
    draws from ``rng`` follow the reference (meshes.py:108-141)."""
    if isinstance(shape, Box):
        return make_box_mesh(shape.half_extents).sample_surface(n, rng)
    if not isinstance(shape, (Sphere, Capsule)):
        raise ValidationError(f"unknown primitive {type(shape).__name__}")
    d = _unit_normals(rng, n)
    if isinstance(shape, Sphere):
        return shape.center + shape.radius * d
    r, h, k = shape.radius, shape.half_length, shape.axis
    t = rng.uniform(-h, h, size=n)
    along = d @ k
    across = d - along[:, None] * k
    cap = (rng.random(n) < (2 * r / (2 * r + 2 * h)))[:, None]
    on_caps = np.sign(along)[:, None] * h * k + r * d
    on_side = t[:, None] * k + r * across / np.maximum(np.linalg.norm(across, axis=-1, keepdims=True), 1e-12)
    return np.where(cap, on_caps, on_side)


def load_stl(path) -> TriangleMesh:
    """STL, ASCII ("solid ... facet ... vertex x y z") or binary (80-byte
    header, uint32 count, 50-byte facets); vertices deduplicated."""
    data = open(path, "rb").read()
    if data.startswith(b"solid") and b"facet" in data[:2048]:
        words = (ln.split() for ln in data.decode("ascii", "replace").splitlines())
        xyz = [[float(t) for t in w[1:]] for w in words if len(w) == 4 and w[0] == "vertex"]
        return _from_soup(np.float64(xyz).reshape(-1, 3, 3))
    if len(data) < 84:
        raise ValidationError(f"{path}: truncated STL")
    n = int.from_bytes(data[80:84], "little")
    if len(data) < 84 + 50 * n:
        raise ValidationError(f"{path}: STL facet data truncated")
    facets = np.frombuffer(data, dtype=np.uint8, count=50 * n, offset=84).reshape(n, 50)
    return _from_soup(facets[:, 12:48].copy().view("<f4").reshape(n, 3, 3).astype(np.float64))


def load_obj(path) -> TriangleMesh:
    """OBJ 'v' and 'f' records; polygons are fan-triangulated, 'v/t/n' indices accepted."""
    verts, faces = [], []
    for words in (ln.split() for ln in open(path)):
        if words[:1] == ["v"]:
            verts.append([float(t) for t in words[1:4]])
        elif words[:1] == ["f"]:
            ring = [int(t.split("/")[0]) - 1 for t in words[1:]]
            faces.extend(zip([ring[0]] * (len(ring) - 2), ring[1:-1], ring[2:]))
    return TriangleMesh(np.float64(verts), np.int64(faces))


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
