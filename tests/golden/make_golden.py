"""Generate the golden fixtures under tests/golden/ by running the REAL reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Every array stored here comes out of the reference package's own public
functions (``/root/reference/pkg/src/linksdf``) on seeded inputs from
``paper_2309_12543_b200.scenarios``; the argmin outputs use the reference's own
gather (``query.py:146``) plus the SURVEY.md Appendix-B tie/clamp rule, since
the reference never returns an argmin.  The GPU box has no reference: the
GPU parity tests read these files instead.
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import linksdf as ref  # noqa: E402  (reference, read-only)
from linksdf.robot import LinkPoseBatch  # noqa: E402

from paper_2309_12543_b200 import scenarios  # noqa: E402


def _robot(doc):
    tmp = Path(tempfile.mkdtemp()) / f"{doc['name']}.json"
    tmp.write_text(json.dumps(doc))
    return ref.RobotModel.from_json(tmp)


def _argmin(batch, fields, obstacles):
    """Appendix-B argmin on top of the reference gather."""
    d = ref.query_min_distances(batch, obstacles)
    C = batch.n_configs
    link = np.full(C, -1, np.int32)
    voxel = np.full(C, -1, np.int32)
    if obstacles.n_occupied == 0:
        return d, link, voxel
    ix, iy, iz = obstacles.indices.T
    g = batch.values[:, ix, iy, iz]
    best = g.argmin(axis=1)
    clamp = np.float32(batch.d_far_global)
    by_c = {}
    for c, li, f in fields:
        by_c.setdefault(c, []).append((li, f))
    for c in range(C):
        if d[c] == clamp:
            continue
        voxel[c] = best[c]
        v = obstacles.indices[best[c]]
        for li, f in sorted(by_c[c], key=lambda t: t[0]):
            rel = v - f.anchor
            w = np.asarray(f.window_dims)
            if np.all(rel >= 0) and np.all(rel < w) and f.values[tuple(rel)] == d[c]:
                link[c] = li
                break
    return d, link, voxel


def scene(doc, q, points, env_extent, env_res, e_r, r_r, store_grids, store_batch,
          store_windows):
    robot = _robot(doc)
    grid = ref.EnvGrid(env_extent, env_res)
    poses_all = ref.forward_kinematics_batch(robot, ref.ConfigBatch(q))
    gl = [i for i, l in enumerate(robot.links) if l.geometry is not None]
    sdfs = [ref.build_link_sdf(robot.links[i].geometry, e_r, r_r, link_id=i) for i in gl]
    poses = LinkPoseBatch(rotations=poses_all.rotations[:, gl],
                          translations=poses_all.translations[:, gl])
    window = ref.WindowGeometry.build(e_r, grid)
    provider = ref.ExactTransformProvider(window)
    fields = list(ref.place_links_batch(sdfs, poses, grid, provider))
    d_far_global = min(s.d_far for s in sdfs)
    batch = ref.assemble_robot_sdfs(((c, f) for c, _, f in fields), grid, len(q), d_far_global)
    obstacles = ref.voxelize_pointcloud(points, grid)
    d, link, voxel = _argmin(batch, fields, obstacles)
    per_link = ref.per_link_min_distances(iter(fields), obstacles, len(q), len(gl), d_far_global)
    out = dict(
        robot_json=np.frombuffer(json.dumps(doc).encode(), dtype=np.uint8),
        q=q, points=points, env_extent=np.float64(env_extent), env_res=np.float64(env_res),
        e_r=np.float64(e_r), r_r=np.float64(r_r),
        R=poses_all.rotations, T=poses_all.translations, geometry_links=np.int64(gl),
        anchors=np.stack([np.stack([f.anchor for c, li, f in fields if c == cc])
                          for cc in range(len(q))]),
        indices=obstacles.indices, n_points=np.int64(obstacles.n_points),
        n_dropped=np.int64(obstacles.n_dropped),
        d=d, link=link, voxel=voxel, per_link=per_link,
        d_far_global=np.float64(d_far_global),
    )
    # anchors above were collected in yield order (link-major); re-sort per (c, l)
    anc = np.zeros((len(q), len(gl), 3), np.int64)
    win = None
    if store_windows:
        wd = window.dims
        win = np.zeros((len(q), len(gl)) + tuple(wd), np.float32)
    for c, li, f in fields:
        anc[c, li] = f.anchor
        if win is not None:
            win[c, li] = f.values
    out["anchors"] = anc
    if win is not None:
        out["windows"] = win
    if store_grids:
        out["grids"] = np.stack([np.asarray(s.values) for s in sdfs])
    else:
        # spot checks of every grid: 4096 fixed cells plus a full-grid checksum
        rng = np.random.default_rng(99)
        S = sdfs[0].dims
        cells = rng.integers(0, S, size=(4096, 3))
        out["grid_cells"] = cells
        out["grid_samples"] = np.stack([np.asarray(s.values)[cells[:, 0], cells[:, 1], cells[:, 2]]
                                        for s in sdfs])
        out["grid_sums"] = np.float64([np.asarray(s.values, dtype=np.float64).sum() for s in sdfs])
    if store_batch:
        out["batch"] = np.asarray(batch.values)
    return out


def known_answer():
    """SURVEY.md Appendix B scene (two identity-rotation links, exact tie)."""
    grid = ref.EnvGrid(1.0, 0.1)
    sph = ref.build_link_sdf(ref.Sphere(0.12), 0.3, 0.01, link_id=0)
    box = ref.build_link_sdf(ref.Box([0.05, 0.05, 0.05]), 0.3, 0.01, link_id=1)
    rot = np.broadcast_to(np.eye(3), (2, 2, 3, 3)).copy()
    trn = np.float64([[[0.05, 0.05, 0.05], [0.45, 0.05, 0.05]],
                      [[-0.35, 0.05, 0.05], [0.05, 0.05, 0.05]]])
    poses = LinkPoseBatch(rotations=rot, translations=trn)
    window = ref.WindowGeometry.build(0.3, grid)
    fields = list(ref.place_links_batch([sph, box], poses, grid, ref.ExactTransformProvider(window)))
    batch = ref.assemble_robot_sdfs(((c, f) for c, _, f in fields), grid, 2, 0.3)
    out = dict(R=rot, T=trn, grids=np.stack([np.asarray(sph.values), np.asarray(box.values)]))
    sets = {"tie": [[12, 10, 10], [8, 10, 10]], "far": [[0, 0, 0], [19, 19, 19]], "empty": []}
    for name, idx in sets.items():
        idx = np.asarray(idx, np.int64).reshape(-1, 3)
        if len(idx):
            idx = np.unique(idx, axis=0)
        obs = ref.ObstacleVoxelSet(indices=idx, grid=grid, n_points=len(idx), n_dropped=0)
        d, link, voxel = _argmin(batch, fields, obs)
        out[f"{name}_indices"] = idx
        out[f"{name}_d"], out[f"{name}_link"], out[f"{name}_voxel"] = d, link, voxel
    return out


def builds():
    """Link-SDF builds: every primitive kind plus signed and open meshes."""
    out = {}
    prims = {
        "sphere": {"type": "sphere", "radius": 0.11, "center": [0.01, -0.02, 0.015]},
        "capsule_z": {"type": "capsule", "radius": 0.06, "half_length": 0.08},
        "capsule_tilt": {"type": "capsule", "radius": 0.05, "half_length": 0.07,
                         "axis": [0.3, -0.5, 0.8]},
        "box": {"type": "box", "half_extents": [0.11, 0.07, 0.09]},
    }
    for name, g in prims.items():
        geo = {"sphere": lambda g: ref.Sphere(g["radius"], center=g.get("center", (0, 0, 0))),
               "capsule": lambda g: ref.Capsule(g["radius"], g["half_length"],
                                                axis=g.get("axis", (0, 0, 1))),
               "box": lambda g: ref.Box(g["half_extents"])}[g["type"]](g)
        s = ref.build_link_sdf(geo, 0.2, 0.01, link_id=0)
        out[f"prim_{name}"] = np.asarray(s.values)
        out[f"prim_{name}_json"] = np.frombuffer(json.dumps(g).encode(), dtype=np.uint8)
    ico = ref.make_icosphere(0.15, subdivisions=1)
    box = ref.make_box_mesh([0.1, 0.07, 0.12])
    tilt = ref.TriangleMesh(box.vertices @ ref.robot.rpy_matrix(0.3, -0.2, 0.5).T, box.triangles)
    open_mesh = ref.TriangleMesh(box.vertices, box.triangles[:-2])
    for name, m, e, r in (("ico", ico, 0.2, 0.0125), ("box", box, 0.2, 0.0125),
                          ("tiltbox", tilt, 0.2, 0.0125), ("open", open_mesh, 0.2, 0.025)):
        s = ref.build_link_sdf(m, e, r, link_id=0)
        out[f"mesh_{name}"] = np.asarray(s.values)
        out[f"mesh_{name}_V"] = m.vertices
        out[f"mesh_{name}_F"] = m.triangles
        out[f"mesh_{name}_er"] = np.float64([e, r])
    return out


def mlp():
    """TinyMlp inference on a W=6 window with random weights."""
    grid = ref.EnvGrid(1.0, 0.1)
    window = ref.WindowGeometry.build(0.3, grid)
    model = ref.TinyMlp.random(window.n_masked, hidden=32, seed=5)
    rng = np.random.default_rng(11)
    R = ref.sample_rotations(rng, 40)
    dt = rng.uniform(-0.05, 0.05, size=(40, 3))
    return dict(w1=model.w1, b1=model.b1, w2=model.w2, b2=model.b2, R=R, dt=dt,
                predict=model.predict(R),
                infer=ref.infer_grid_transform(model, R, dt, 0.3),
                exact=ref.grid_transform_exact(R, dt, 0.3, window.masked_points),
                masked_points=window.masked_points)


def trilinear_cases():
    rng = np.random.default_rng(21)
    s = ref.build_link_sdf(ref.Capsule(0.06, 0.08), 0.32, 0.02, link_id=0)
    pts = rng.uniform(-0.36, 0.36, size=(20000, 3))
    return dict(values=np.asarray(s.values), extent=np.float64(0.32), res=np.float64(0.02),
                pts=pts, out=ref.trilinear_sample(s, pts))


def main():
    scenes = {}
    doc = scenarios.ARM6G
    q1 = scenarios.random_configs(doc, 64, seed=1)
    p1 = scenarios.human_cloud(10_000, seed=1)
    scenes["scene_c1"] = scene(doc, q1, p1, 1.0, 0.04, 0.32, 0.02, store_grids=True,
                               store_batch=False, store_windows=False)
    q2 = scenarios.random_configs(doc, 24, seed=2)
    p2 = scenarios.human_cloud(30_000, seed=2)
    scenes["scene_c2"] = scene(doc, q2, p2, 1.0, 0.04, 0.32, 0.01, store_grids=False,
                               store_batch=False, store_windows=False)
    q3 = scenarios.random_configs(doc, 12, seed=3)
    p3 = scenarios.human_cloud(3_000, seed=3)
    scenes["scene_small"] = scene(doc, q3, p3, 1.0, 0.1, 0.3, 0.02, store_grids=True,
                                  store_batch=True, store_windows=True)
    doc7 = scenarios.ARM7G
    q4 = scenarios.random_configs(doc7, 16, seed=4)
    p4 = scenarios.crowd_cloud(3, 4000, seed=4)
    scenes["scene_arm7"] = scene(doc7, q4, p4, 1.0, 0.04, 0.32, 0.02, store_grids=False,
                                 store_batch=False, store_windows=False)
    for name, arrays in scenes.items():
        np.savez_compressed(HERE / f"{name}.npz", **arrays)
    np.savez_compressed(HERE / "known_answer.npz", **known_answer())
    np.savez_compressed(HERE / "builds.npz", **builds())
    np.savez_compressed(HERE / "mlp.npz", **mlp())
    np.savez_compressed(HERE / "trilinear.npz", **trilinear_cases())
    for p in sorted(HERE.glob("*.npz")):
        print(f"{p.name}: {p.stat().st_size / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
