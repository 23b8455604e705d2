"""CPU oracle for the batched link-SDF distance checker — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's hot path
(``/root/reference/pkg/src/linksdf``, "linksdf" 0.1.0).  It exists so that the
CUDA product path can be checked on the GPU box, where the reference itself is
absent.  Rules:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` leg may import it;
* the product package ``paper_2309_12543_b200`` never imports it;
* every function cites the reference ``file:line`` it restates and repeats the
  same numpy operations in the same order, so on the same numpy/OpenBLAS build
  its results are bit-identical to the reference's.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(importable in the build container) on seeded scenes and stores inputs and
outputs under ``tests/golden/*.npz``; ``tests/test_oracle.py`` checks this
restatement against those fixtures bit-for-bit (FK to 1e-12, the reference's
own bar).  The argmin (link, point) outputs are the SURVEY.md Appendix-B
restatement on top of the reference's own gather (``query.py:146``) — the
reference never returns an argmin, so those are pinned on that construction.

Data conventions match the reference: link grids are (nx, ny, nz) float32
arrays indexed [ix, iy, iz] and stored x-fastest; environment voxel indices
are (N, 3) int64 sorted lexicographically; rotations are (C, L, 3, 3) float64.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# Robot description → flat chain (robot.py:24-46, 178-239)
# ---------------------------------------------------------------------------


def rpy(roll, pitch, yaw):
    """robot.py:24-32 — Rz @ Ry @ Rx."""
    cr, sr, cp, sp, cy, sy = (np.cos(roll), np.sin(roll), np.cos(pitch),
                              np.sin(pitch), np.cos(yaw), np.sin(yaw))
    rz = np.array([[cy, -sy, 0.0], [sy, cy, 0.0], [0.0, 0.0, 1.0]])
    ry = np.array([[cp, 0.0, sp], [0.0, 1.0, 0.0], [-sp, 0.0, cp]])
    rx = np.array([[1.0, 0.0, 0.0], [0.0, cr, -sr], [0.0, sr, cr]])
    return rz @ ry @ rx


def rodrigues(axis, angles):
    """robot.py:35-46 — c*I + s*[k]x + (1-c)*k k^T for a vector of angles."""
    k = np.asarray(axis, dtype=np.float64)
    angles = np.asarray(angles, dtype=np.float64)
    skew = np.array([[0.0, -k[2], k[1]], [k[2], 0.0, -k[0]], [-k[1], k[0], 0.0]])
    outer = np.outer(k, k)
    c = np.cos(angles)[..., None, None]
    s = np.sin(angles)[..., None, None]
    return c * np.eye(3) + s * skew + (1.0 - c) * outer


def _origin(obj):
    if obj is None:
        return np.eye(3), np.zeros(3)
    return rpy(*obj.get("rpy", [0.0, 0.0, 0.0])), np.asarray(
        obj.get("xyz", [0.0, 0.0, 0.0]), dtype=np.float64)


def chain_from_doc(doc: dict) -> list[dict]:
    """Flatten a robot JSON document into parents-first link records."""
    joints = {j["name"]: j for j in doc.get("joints", [])}
    actuated = [j["name"] for j in doc.get("joints", []) if j["type"] != "fixed"]
    names = [l["name"] for l in doc["links"]]
    out = []
    for link in doc["links"]:
        rec = {"name": link["name"], "geometry": link.get("geometry")}
        rec["link_R"], rec["link_t"] = _origin(link.get("origin"))
        pj = link.get("parent_joint")
        if pj is None:
            rec["kind"] = "base"
        else:
            j = joints[pj]
            rec["kind"] = j["type"]
            rec["parent"] = names.index(j["parent_link"])
            rec["joint_R"], rec["joint_t"] = _origin(j.get("origin"))
            rec["axis"] = np.asarray(j.get("axis", [0.0, 0.0, 1.0]), dtype=np.float64)
            rec["col"] = actuated.index(pj) if j["type"] != "fixed" else -1
        out.append(rec)
    return out


def limits_from_doc(doc: dict) -> np.ndarray:
    rows = []
    for j in doc.get("joints", []):
        if j["type"] == "fixed":
            continue
        pos = j.get("limits", {}).get("position")
        rows.append(pos if pos else (-np.inf, np.inf))
    return np.asarray(rows, dtype=np.float64).reshape(-1, 2)


def limit_violations(doc: dict, q: np.ndarray) -> list[tuple[int, int]]:
    """robot.py:291-302."""
    lim = limits_from_doc(doc)
    bad = (q < lim[:, 0]) | (q > lim[:, 1])
    cs, js = np.nonzero(bad)
    return list(zip(cs.tolist(), js.tolist()))


def fk(chain: list[dict], q: np.ndarray):
    """robot.py:305-347 — batched FK, fp64, same operation order."""
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    n = q.shape[0]
    R = np.empty((n, len(chain), 3, 3))
    T = np.empty((n, len(chain), 3))
    for li, rec in enumerate(chain):
        if rec["kind"] == "base":
            rj = np.broadcast_to(np.eye(3), (n, 3, 3))
            tj = np.zeros((n, 3))
        else:
            rp = R[:, rec["parent"]]
            tp = T[:, rec["parent"]]
            ro, to = rec["joint_R"], rec["joint_t"]
            if rec["kind"] == "revolute":
                rl = ro @ rodrigues(rec["axis"], q[:, rec["col"]])
                tl = np.broadcast_to(to, (n, 3))
            elif rec["kind"] == "prismatic":
                rl = np.broadcast_to(ro, (n, 3, 3))
                tl = to + np.outer(q[:, rec["col"]], ro @ rec["axis"])
            else:
                rl = np.broadcast_to(ro, (n, 3, 3))
                tl = np.broadcast_to(to, (n, 3))
            rj = rp @ rl
            tj = tp + np.einsum("cij,cj->ci", rp, tl)
        R[:, li] = rj @ rec["link_R"]
        T[:, li] = tj + np.einsum("cij,j->ci", rj, rec["link_t"])
    return R, T


def geometry_links(chain) -> list[int]:
    """bench.py:128 — links carrying collision geometry, in declaration order."""
    return [i for i, rec in enumerate(chain) if rec["geometry"] is not None]


# ---------------------------------------------------------------------------
# Environment grid, alignment, window tables (grids.py:49-113, placement.py:29-145)
# ---------------------------------------------------------------------------


class Env:
    """grids.py:49-90 — extent/resolution/dims plus the index helpers."""

    def __init__(self, extent, resolution):
        self.extent = np.broadcast_to(np.asarray(extent, dtype=np.float64), (3,)).copy()
        self.resolution = np.broadcast_to(np.asarray(resolution, dtype=np.float64), (3,)).copy()
        self.dims = np.rint(2.0 * self.extent / self.resolution).astype(np.int64)

    def centers(self, idx):
        return -self.extent + (np.asarray(idx, dtype=np.float64) + 0.5) * self.resolution


def window_width(e_r: float, env: Env) -> np.ndarray:
    """placement.py:29-44 (validation omitted: callers pass valid shapes)."""
    ratio = 2.0 * np.broadcast_to(np.float64(e_r), (3,)) / env.resolution
    return np.rint(ratio).astype(np.int64)


def align(T, env: Env, e_r: float):
    """placement.py:60-99 — (anchor int64, delta_t f64) with the face guard."""
    w = window_width(e_r, env)
    pos = np.asarray(T, dtype=np.float64).reshape(-1, 3)
    j = np.floor((pos + env.extent) / env.resolution).astype(np.int64)
    delta = pos - env.centers(j)
    half = 0.5 * env.resolution
    slack = 32.0 * np.finfo(np.float64).eps * np.maximum(env.extent, 1.0)
    j += (delta >= half).astype(np.int64)
    j -= (delta < -half - slack).astype(np.int64)
    delta = pos - env.centers(j)
    anchor = j - w // 2
    no_overlap = np.any((anchor >= env.dims) | (anchor + w <= 0), axis=-1)
    return anchor, delta, no_overlap


def window_points(e_r: float, env: Env) -> np.ndarray:
    """placement.py:112-125 — normalized window cell centres, x-fastest."""
    w = window_width(e_r, env)
    axes = [(np.arange(w[a]) - w[a] // 2) * env.resolution[a] / e_r for a in range(3)]
    zz, yy, xx = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    return np.stack([xx, yy, zz], axis=-1).reshape(-1, 3)


def window_mask(e_r: float, env: Env) -> np.ndarray:
    """placement.py:128-145 — ball keep-mask, shape (W, W, W) indexed [x, y, z]."""
    w = window_width(e_r, env)
    axes = [(np.arange(w[a]) - w[a] // 2) * env.resolution[a] for a in range(3)]
    xx, yy, zz = np.meshgrid(axes[0], axes[1], axes[2], indexing="ij")
    return xx * xx + yy * yy + zz * zz < e_r * e_r * (1.0 - 1e-12)


def transform_exact(R, dt, e_r, points):
    """placement.py:148-169 — G = P R + (-(dt/e_r) R), row-vector form."""
    R = np.asarray(R, dtype=np.float64).reshape(-1, 3, 3)
    dt = np.asarray(dt, dtype=np.float64).reshape(-1, 3)
    g = np.matmul(points[None], R)
    g += (-np.einsum("bj,bjk->bk", dt / e_r, R))[:, None, :]
    return g


# ---------------------------------------------------------------------------
# Trilinear sampling (grids.py:155-191)
# ---------------------------------------------------------------------------


def trilinear(values: np.ndarray, extent, resolution, pts) -> np.ndarray:
    extent = np.broadcast_to(np.asarray(extent, dtype=np.float64), (3,))
    resolution = np.broadcast_to(np.asarray(resolution, dtype=np.float64), (3,))
    dims = np.asarray(values.shape, dtype=np.int64)
    p = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    u = (p + extent) / resolution - 0.5
    top = (dims - 1).astype(np.float64)
    inside = np.all((u >= 0.0) & (u <= top), axis=-1)
    uc = np.clip(u, 0.0, top)
    i0 = np.minimum(uc.astype(np.int64), dims - 2)
    f = (uc - i0).astype(np.float32)
    flat = np.asarray(values, dtype=np.float32).ravel(order="F")
    nx, ny = int(dims[0]), int(dims[1])
    b = i0[:, 0] + nx * (i0[:, 1] + ny * i0[:, 2])
    sy, sz = nx, nx * ny
    fx, fy, fz = f[:, 0], f[:, 1], f[:, 2]
    gx, gy, gz = 1.0 - fx, 1.0 - fy, 1.0 - fz
    c00 = flat[b] * gx + flat[b + 1] * fx
    c10 = flat[b + sy] * gx + flat[b + 1 + sy] * fx
    c01 = flat[b + sz] * gx + flat[b + 1 + sz] * fx
    c11 = flat[b + sy + sz] * gx + flat[b + 1 + sy + sz] * fx
    out = (c00 * gy + c10 * fy) * gz + (c01 * gy + c11 * fy) * fz
    d_far = float(np.min(extent))
    return np.where(inside, out, np.float32(d_far)).astype(np.float32)


# ---------------------------------------------------------------------------
# Placement + assembly + query (placement.py:267-313, query.py:61-176)
# ---------------------------------------------------------------------------


def place_windows(grids, grid_extents, grid_res, R, T, env: Env, e_r: float, chunk=8):
    """placement.py:267-313 — every (c, l) window, dense (C, L, W, W, W) f32.

    ``grids[l]`` is the (S, S, S) f32 link SDF; masked cells carry the link's
    far sentinel.  Returns (windows, anchors (C, L, 3) int64).
    """
    C, L = R.shape[:2]
    w = window_width(e_r, env)
    pts = window_points(e_r, env)
    mask_f = window_mask(e_r, env).ravel(order="F")
    kept = pts[mask_f]
    anchor, delta, _ = align(T.reshape(-1, 3), env, e_r)
    anchor = anchor.reshape(C, L, 3)
    delta = delta.reshape(C, L, 3)
    out = np.empty((C, L, int(np.prod(w))), dtype=np.float32)
    for li in range(L):
        ext = np.broadcast_to(np.asarray(grid_extents[li], dtype=np.float64), (3,))
        d_far = np.float32(float(np.min(ext)))
        for c0 in range(0, C, chunk):
            c1 = min(c0 + chunk, C)
            g = transform_exact(R[c0:c1, li], delta[c0:c1, li], e_r, kept)
            s = trilinear(grids[li], ext, grid_res[li], (g * e_r).reshape(-1, 3))
            blk = np.full((c1 - c0, out.shape[2]), d_far, dtype=np.float32)
            blk[:, mask_f] = s.reshape(c1 - c0, -1)
            out[c0:c1, li] = blk
    windows = out.reshape(C, L, int(w[2]), int(w[1]), int(w[0])).transpose(0, 1, 4, 3, 2)
    return windows, anchor


def assemble(windows, anchors, env: Env, d_far_global: float) -> np.ndarray:
    """query.py:61-103 — min-merge into dense (C, nx, ny, nz) f32."""
    C, L = windows.shape[:2]
    dims = env.dims
    out = np.full((C,) + tuple(dims), np.float32(d_far_global), dtype=np.float32)
    w = np.asarray(windows.shape[2:], dtype=np.int64)
    for c in range(C):
        for li in range(L):
            k = anchors[c, li]
            lo = np.maximum(k, 0)
            hi = np.minimum(k + w, dims)
            if np.any(lo >= hi):
                continue
            src = windows[c, li, lo[0] - k[0]:hi[0] - k[0], lo[1] - k[1]:hi[1] - k[1],
                          lo[2] - k[2]:hi[2] - k[2]]
            dst = out[c, lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]
            np.minimum(dst, src, out=dst)
    return out


def voxelize(points, env: Env):
    """query.py:106-125 + grids.py:93-113 — (indices, n_points, n_dropped)."""
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    inside = np.all((p >= -env.extent) & (p < env.extent), axis=-1)
    kept = p[inside]
    if len(kept):
        idx = np.floor((kept + env.extent) / env.resolution).astype(np.int64)
        np.clip(idx, 0, env.dims - 1, out=idx)
        idx = np.unique(idx, axis=0)
    else:
        idx = np.empty((0, 3), dtype=np.int64)
    return idx, len(p), int(len(p) - inside.sum())


def query_min(batch: np.ndarray, indices: np.ndarray, d_far_global: float):
    """query.py:128-150 — gather + min; empty set → far sentinel."""
    if len(indices) == 0:
        return np.full(batch.shape[0], np.float32(d_far_global), dtype=np.float32)
    g = batch[:, indices[:, 0], indices[:, 1], indices[:, 2]]
    return g.min(axis=1)


def per_link_min(windows, anchors, indices, d_far_links, d_far_global):
    """query.py:153-176 — (C, L) per-link minima."""
    C, L = windows.shape[:2]
    w = np.asarray(windows.shape[2:], dtype=np.int64)
    out = np.full((C, L), np.float32(d_far_global), dtype=np.float32)
    for c in range(C):
        for li in range(L):
            rel = indices - anchors[c, li]
            ok = np.all((rel >= 0) & (rel < w), axis=-1)
            lim = min(float(d_far_links[li]), float(out[c, li]))
            if np.any(ok):
                vals = windows[c, li][rel[ok, 0], rel[ok, 1], rel[ok, 2]]
                lim = min(lim, float(vals.min()))
            out[c, li] = lim
    return out


def argmin_oracle(batch, windows, anchors, indices, d_far_global):
    """(d, link, voxel) with the clamp/empty rules.

    voxel = first occurrence of the minimum in the reference gather order
    (``query.py:146``); link = lowest link whose window covers that voxel with
    exactly that value; d == f32(d_far_global) → link = voxel = -1.
    """
    C, L = windows.shape[:2]
    d = query_min(batch, indices, d_far_global)
    link = np.full(C, -1, dtype=np.int32)
    voxel = np.full(C, -1, dtype=np.int32)
    if len(indices) == 0:
        return d, link, voxel
    g = batch[:, indices[:, 0], indices[:, 1], indices[:, 2]]
    best = g.argmin(axis=1)
    w = np.asarray(windows.shape[2:], dtype=np.int64)
    clamp = np.float32(d_far_global)
    for c in range(C):
        if d[c] == clamp:
            continue
        v = indices[best[c]]
        voxel[c] = best[c]
        for li in range(L):
            rel = v - anchors[c, li]
            if np.all(rel >= 0) and np.all(rel < w):
                if windows[c, li][rel[0], rel[1], rel[2]] == d[c]:
                    link[c] = li
                    break
    return d, link, voxel


# ---------------------------------------------------------------------------
# Link-SDF build (meshes.py:64-82, 144-371)
# ---------------------------------------------------------------------------


def primitive_sdf(geom: dict, pts) -> np.ndarray:
    """meshes.py:64-82 with the JSON geometry dict (robot.py:223-239)."""
    p = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    kind = geom["type"]
    if kind == "sphere":
        c = np.asarray(geom.get("center", (0, 0, 0)), dtype=np.float64)
        return np.linalg.norm(p - c, axis=-1) - float(geom["radius"])
    if kind == "capsule":
        ax = np.asarray(geom.get("axis", (0.0, 0.0, 1.0)), dtype=np.float64)
        ax = ax / np.linalg.norm(ax)
        hl = float(geom["half_length"])
        t = np.clip(p @ ax, -hl, hl)
        return np.linalg.norm(p - t[:, None] * ax, axis=-1) - float(geom["radius"])
    if kind == "box":
        q = np.abs(p) - np.asarray(geom["half_extents"], dtype=np.float64)
        return np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(np.max(q, axis=-1), 0.0)
    raise ValueError(kind)


def _closest_sq(p, a, b, c):
    """meshes.py:144-214 — Voronoi-region closest point, squared distance (n, t)."""
    ab, ac, bc = b - a, c - a, c - b
    ap = p[:, None, :] - a[None]
    bp = p[:, None, :] - b[None]
    cp = p[:, None, :] - c[None]
    d1 = np.einsum("ntj,tj->nt", ap, ab)
    d2 = np.einsum("ntj,tj->nt", ap, ac)
    d3 = np.einsum("ntj,tj->nt", bp, ab)
    d4 = np.einsum("ntj,tj->nt", bp, ac)
    d5 = np.einsum("ntj,tj->nt", cp, ab)
    d6 = np.einsum("ntj,tj->nt", cp, ac)
    va = d3 * d6 - d5 * d4
    vb = d5 * d2 - d1 * d6
    vc = d1 * d4 - d3 * d2
    with np.errstate(divide="ignore", invalid="ignore"):
        t_ab = np.nan_to_num(d1 / (d1 - d3))
        t_ac = np.nan_to_num(d2 / (d2 - d6))
        t_bc = np.nan_to_num((d4 - d3) / ((d4 - d3) + (d5 - d6)))
    denom = va + vb + vc
    denom = np.where(denom == 0, 1.0, denom)
    v = vb / denom
    w = vc / denom
    shape = ap.shape
    cands = [
        ((d1 <= 0) & (d2 <= 0), np.broadcast_to(a[None], shape)),
        ((d3 >= 0) & (d4 <= d3), np.broadcast_to(b[None], shape)),
        ((vc <= 0) & (d1 >= 0) & (d3 <= 0), a[None] + t_ab[..., None] * ab[None]),
        ((d6 >= 0) & (d5 <= d6), np.broadcast_to(c[None], shape)),
        ((vb <= 0) & (d2 >= 0) & (d6 <= 0), a[None] + t_ac[..., None] * ac[None]),
        ((va <= 0) & ((d4 - d3) >= 0) & ((d5 - d6) >= 0), b[None] + t_bc[..., None] * bc[None]),
        (np.ones(d1.shape, dtype=bool), a[None] + v[..., None] * ab[None] + w[..., None] * ac[None]),
    ]
    closest = np.empty_like(ap)
    done = np.zeros(d1.shape, dtype=bool)
    for m, val in cands:
        m = m & ~done
        closest[m] = val[m]
        done |= m
    diff = p[:, None, :] - closest
    return np.einsum("ntj,ntj->nt", diff, diff)


RAY_DIRECTIONS = np.float64([
    [0.577350269, 0.577350269, 0.577350269],
    [0.267261242, 0.534522484, 0.801783726],
    [-0.455842306, 0.569802882, 0.683763459],
    [0.816496581, -0.408248290, 0.408248290],
])  # meshes.py:249-256


def _crossings(p, a, b, c, direction):
    """meshes.py:259-289 — (hit counts, suspect) along one direction."""
    e1, e2 = b - a, c - a
    h = np.cross(direction, e2)
    det = np.einsum("tj,tj->t", e1, h)
    parallel = np.abs(det) < 1e-12
    det_safe = np.where(parallel, 1.0, det)
    s = p[:, None, :] - a[None]
    u = np.einsum("ntj,tj->nt", s, h) / det_safe
    qv = np.cross(s, e1[None])
    v = np.einsum("ntj,j->nt", qv, direction) / det_safe
    t = np.einsum("ntj,tj->nt", qv, e2) / det_safe
    hit = (~parallel) & (u >= 0) & (v >= 0) & (u + v <= 1) & (t > 0)
    eps = 1e-9
    near = hit & ((u < eps) | (v < eps) | (u + v > 1 - eps) | (np.abs(t) < eps))
    return hit.sum(axis=1), near.any(axis=1)


def mesh_sdf(vertices, triangles, pts, signed=True, chunk=4096):
    """meshes.py:217-329 — exact distance, ray-parity sign (no prefilter:
    the reference's centroid prefilter only drops triangles that cannot win)."""
    V = np.asarray(vertices, dtype=np.float64)
    F = np.asarray(triangles, dtype=np.int64)
    a, b, c = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    p = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.empty(len(p))
    for s0 in range(0, len(p), chunk):
        blk = p[s0:s0 + chunk]
        d = np.sqrt(_closest_sq(blk, a, b, c).min(axis=1))
        if signed:
            inside = np.zeros(len(blk), dtype=bool)
            rem = np.arange(len(blk))
            for direction in RAY_DIRECTIONS:
                cnt, sus = _crossings(blk[rem], a, b, c, direction)
                ok = ~sus
                inside[rem[ok]] = cnt[ok] % 2 == 1
                rem = rem[sus]
                if len(rem) == 0:
                    break
            d = np.where(inside, -d, d)
        out[s0:s0 + chunk] = d
    return out


def cell_centers(extent, resolution):
    extent = np.broadcast_to(np.asarray(extent, dtype=np.float64), (3,))
    resolution = np.broadcast_to(np.asarray(resolution, dtype=np.float64), (3,))
    dims = np.rint(2.0 * extent / resolution).astype(np.int64)
    return [-extent[a] + (np.arange(dims[a]) + 0.5) * resolution[a] for a in range(3)]


def build_grid(geom: dict, extent, resolution, mesh=None) -> np.ndarray:
    """meshes.py:332-371 — dense (nx, ny, nz) f32 grid of exact distances."""
    axes = cell_centers(extent, resolution)
    gx, gy, gz = np.meshgrid(*axes, indexing="ij")
    centers = np.stack([gx, gy, gz], axis=-1).reshape(-1, 3)
    if mesh is not None:
        d = mesh_sdf(mesh[0], mesh[1], centers, signed=mesh[2])
    else:
        d = primitive_sdf(geom, centers)
    return d.reshape(gx.shape).astype(np.float32)


# ---------------------------------------------------------------------------
# TinyMlp inference (approx.py:123-130, 292-306)
# ---------------------------------------------------------------------------


def mlp_predict(w1, b1, w2, b2, R):
    x = np.asarray(R, dtype=np.float32).reshape(-1, 9)
    h = np.maximum(x @ w1 + b1, 0.0)
    return (h @ w2 + b2).reshape(len(x), -1, 3)


def mlp_transform(w1, b1, w2, b2, R, dt, e_r):
    R = np.asarray(R, dtype=np.float64).reshape(-1, 3, 3)
    g = mlp_predict(w1, b1, w2, b2, R).astype(np.float64)
    return g + (-np.einsum("bj,bjk->bk", np.asarray(dt).reshape(-1, 3) / float(e_r), R))[:, None, :]


# ---------------------------------------------------------------------------
# Whole path: configurations + points → (d, link, voxel)
# ---------------------------------------------------------------------------


def run_pipeline(doc: dict, q, points, env_extent, env_res, e_r, grids, grid_res,
                 return_all=False):
    """FK → placement → assembly → voxelize → query → argmin (bench.py:126-179)."""
    chain = chain_from_doc(doc)
    env = Env(env_extent, env_res)
    R, T = fk(chain, q)
    gl = geometry_links(chain)
    Rg, Tg = R[:, gl], T[:, gl]
    windows, anchors = place_windows(grids, [e_r] * len(gl), grid_res, Rg, Tg, env, e_r)
    d_far_global = float(e_r)
    batch = assemble(windows, anchors, env, d_far_global)
    idx, n_pts, n_drop = voxelize(points, env)
    d, link, voxel = argmin_oracle(batch, windows, anchors, idx, d_far_global)
    if return_all:
        return dict(R=R, T=T, anchors=anchors, windows=windows, batch=batch,
                    indices=idx, n_points=n_pts, n_dropped=n_drop,
                    d=d, link=link, voxel=voxel)
    return d, link, voxel
