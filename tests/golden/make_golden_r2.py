"""Round-2 fixtures from the REAL reference: the benchmarked inputs themselves.

    python tests/golden/make_golden_r2.py        # build container only (/root/reference)

* ``bench_c2.npz`` — BASELINE config 2 exactly as bench.py feeds it: arm6g,
  500 waypoints of ``random_configs(seed)`` against ``cloud_for(CONFIG2, seed)``
  cast to f32 (frames are f32 on disk), seeds 21-24, 64^3 link grids: the
  reference's d plus the Appendix-B argmin (link, voxel) for every waypoint.
* ``bench_c4.npz`` — BASELINE config 4's seed-11 step: 16 waypoints
  (every 4,096th of the 65,536) against the full 1M-point f32 crowd cloud.
* ``builds128.npz`` — config 3 (i): the six arm6g primitives and the
  1,280-triangle icosphere at 128^3 (e_r 0.64, r_r 0.01): reference values at
  a strided subset of cells (every 97th x-fastest cell for primitives, 3,000
  seeded cells for the mesh, where each cell costs 1,280 triangle tests) plus
  the full-grid f64 sums of the primitives.
* ``sphere_c2.npz`` — the covering-sphere comparator (query.py:254-291) on
  config 2's seed-21 input, arm6g with 18 covering spheres.

Inputs are regenerated from ``paper_2309_12543_b200.scenarios`` (seeded numpy);
the fixtures store checksums of them so drift fails loudly.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden as MG  # noqa: E402  (puts the reference on sys.path)

ref = MG.ref
from linksdf.robot import LinkPoseBatch  # noqa: E402

from paper_2309_12543_b200 import scenarios as S  # noqa: E402


def _run(doc, q, pts, shape):
    robot = MG._robot(doc)
    grid = ref.EnvGrid(shape.grid_extent, shape.grid_res)
    poses_all = ref.forward_kinematics_batch(robot, ref.ConfigBatch(q))
    gl = [i for i, l in enumerate(robot.links) if l.geometry is not None]
    sdfs = [ref.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i) for i in gl]
    poses = LinkPoseBatch(rotations=poses_all.rotations[:, gl], translations=poses_all.translations[:, gl])
    window = ref.WindowGeometry.build(shape.link_extent, grid)
    fields = list(ref.place_links_batch(sdfs, poses, grid, ref.ExactTransformProvider(window)))
    d_far = min(s.d_far for s in sdfs)
    batch = ref.assemble_robot_sdfs(((c, f) for c, _, f in fields), grid, len(q), d_far)
    obs = ref.voxelize_pointcloud(pts, grid)
    d, link, voxel = MG._argmin(batch, fields, obs)
    return d, link, voxel, obs.n_occupied, obs.n_dropped


def _digest(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    return np.float64([a.astype(np.float64).sum(), np.abs(a.astype(np.float64)).sum(), a.size])


def bench_c2():
    shape = S.CONFIG2
    out = {}
    for seed in (21, 22, 23, 24):
        q = S.random_configs(shape.robot, shape.n_waypoints, seed=seed)
        pts = S.cloud_for(shape, seed).astype(np.float32)
        d, link, voxel, n_occ, n_drop = _run(shape.robot, q, pts, shape)
        out.update({f"s{seed}_d": d, f"s{seed}_link": link, f"s{seed}_voxel": voxel,
                    f"s{seed}_n_occ": np.int64(n_occ), f"s{seed}_q_digest": _digest(q),
                    f"s{seed}_pts_digest": _digest(pts)})
        print(f"config 2 seed {seed}: N_occ {n_occ}, {np.sum(link >= 0)} waypoints with an obstacle in range")
    return out


def bench_c4():
    shape = S.CONFIG4
    q_all = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    sub = np.arange(0, shape.n_waypoints, 4096)
    pts = S.cloud_for(shape, 11).astype(np.float32)
    d, link, voxel, n_occ, n_drop = _run(shape.robot, q_all[sub], pts, shape)
    print(f"config 4 seed 11: N_occ {n_occ}, dropped {n_drop}")
    return {"sub": sub, "d": d, "link": link, "voxel": voxel, "n_occ": np.int64(n_occ),
            "n_dropped": np.int64(n_drop), "q_digest": _digest(q_all), "pts_digest": _digest(pts)}


def builds128():
    e_r, r_r = 0.64, 0.01
    robot = MG._robot(S.ARM6G)
    out = {}
    rng = np.random.default_rng(128)
    for i, link in enumerate(robot.links):
        if link.geometry is None:
            continue
        s = ref.build_link_sdf(link.geometry, e_r, r_r, link_id=i)
        flat = np.asarray(s.values).ravel(order="F")
        out[f"prim_{link.name}_idx"] = np.arange(0, flat.size, 97, dtype=np.int64)
        out[f"prim_{link.name}"] = flat[::97].copy()
        out[f"prim_{link.name}_sum"] = np.float64(flat.astype(np.float64).sum())
    ico = ref.make_icosphere(0.08, subdivisions=3)
    assert len(ico.triangles) == 1280
    idx = np.sort(rng.choice(128 ** 3, size=3000, replace=False))
    ijk = np.stack(np.unravel_index(idx, (128, 128, 128), order="F"), axis=1)
    centres = -e_r + (ijk + 0.5) * r_r
    out["mesh_idx"] = idx
    out["mesh"] = ref.exact_point_distance(ico, centres, signed=ico.is_watertight).astype(np.float32)
    out["mesh_V"], out["mesh_F"] = ico.vertices, ico.triangles
    return out


ARM6G_SPHERES = {  # covering spheres of the arm6g primitives: capsules by 3 spheres on the axis, box by 1, sphere itself
    "l1": [{"center": [0, 0, z], "radius": 0.07} for z in (-0.06, 0.0, 0.06)],
    "l2": [{"center": [0, 0, z], "radius": 0.06} for z in (-0.08, 0.0, 0.08)],
    "l3": [{"center": [0, 0, z], "radius": 0.05} for z in (-0.07, 0.0, 0.07)],
    "l4": [{"center": [0, 0, z], "radius": 0.045} for z in (-0.05, 0.0, 0.05)],
    "l5": [{"center": [0, 0, 0], "radius": 0.0755}],
    "l6": [{"center": [0, 0, 0], "radius": 0.05}],
}


def sphere_baseline():
    """sphere_baseline_distances (query.py:254-291) on config 2's seed-21 input:
    arm6g with covering spheres, 500 waypoints, the 100k-point human."""
    import json

    shape = S.CONFIG2
    doc = json.loads(json.dumps(shape.robot))
    doc["spheres"] = ARM6G_SPHERES
    robot = MG._robot(doc)
    grid = ref.EnvGrid(shape.grid_extent, shape.grid_res)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=21)
    pts = S.cloud_for(shape, 21).astype(np.float32)
    poses = ref.forward_kinematics_batch(robot, ref.ConfigBatch(q))
    obs = ref.voxelize_pointcloud(pts, grid)
    spheres = ref.SphereRobotModel.from_robot(robot)
    d, st = ref.sphere_baseline_distances(spheres, poses, obs, grid, return_stats=True)
    print(f"sphere baseline: {spheres.n_spheres} spheres, {st['distance_evals']} distance evaluations")
    return {"robot_json": np.frombuffer(json.dumps(doc).encode(), dtype=np.uint8), "d": d,
            "evals": np.int64(st["distance_evals"]), "q_digest": _digest(q), "pts_digest": _digest(pts)}


def main():
    np.savez_compressed(HERE / "sphere_c2.npz", **sphere_baseline())
    np.savez_compressed(HERE / "builds128.npz", **builds128())
    np.savez_compressed(HERE / "bench_c4.npz", **bench_c4())
    np.savez_compressed(HERE / "bench_c2.npz", **bench_c2())
    for n in ("sphere_c2", "builds128", "bench_c4", "bench_c2"):
        p = HERE / f"{n}.npz"
        print(f"{p.name}: {p.stat().st_size / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
