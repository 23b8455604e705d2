"""GPU parity: the CUDA path (through the C ABI) vs the reference goldens and the oracle.

Bars (north_star): FK <= 1e-12 abs; anchors, voxel indices,
argmin link/voxel bit-exact; primitive link grids, windows, assembled fields
and distances bit-exact in fp32 when the poses are the reference's own
(stage isolation); distances from GPU FK within 1e-6 m (the fp64 sin/cos of
the device may differ from the host libm in the last ulp); mesh grids within
1e-5 m; MLP outputs within 1e-5 (normalized).
"""

import json

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu

D_TOL = 1e-6      # m, distances from device FK vs reference FK
MESH_TOL = 1e-5   # m, SURVEY §8c
MLP_TOL = 1e-5    # normalized coordinates


@pytest.fixture(scope="module")
def L():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_12543_b200 as lib

    return lib


def _doc(g):
    return json.loads(bytes(g["robot_json"]).decode())


def _scene(L, g):
    robot = L.RobotModel.from_dict(_doc(g))
    grid = L.EnvGrid(float(g["env_extent"]), float(g["env_res"]))
    e_r, r_r = float(g["e_r"]), float(g["r_r"])
    sdfs = [L.build_link_sdf(robot.links[i].geometry, e_r, r_r, link_id=i) for i in robot.geometry_links]
    window = L.WindowGeometry.build(e_r, grid)
    return robot, grid, sdfs, window


# ----------------------------------------------------------------------------- stage 1


@pytest.mark.parametrize("name", ["scene_c1", "scene_arm7", "scene_small"])
def test_fk_batch(L, name):
    g = golden(name)
    robot = L.RobotModel.from_dict(_doc(g))
    poses = L.forward_kinematics_batch(robot, L.ConfigBatch(g["q"]))
    assert np.abs(poses.rotations - g["R"]).max() <= 1e-12
    assert np.abs(poses.translations - g["T"]).max() <= 1e-12


def test_fk_known_answers(L, tmp_path):
    # test_robot.py:114-155
    doc = {"name": "one", "links": [{"name": "base"}, {"name": "child", "parent_joint": "j",
                                                         "origin": {"xyz": [1, 0, 0]}}],
           "joints": [{"name": "j", "type": "revolute", "parent_link": "base", "axis": [0, 0, 1],
                       "limits": {"position": [-7, 7], "velocity": 1, "acceleration": 1}}]}
    m = L.RobotModel.from_dict(doc)
    p = L.forward_kinematics_batch(m, L.ConfigBatch([[np.pi / 2]]))
    assert np.allclose(p.translations[0, 1], [0, 1, 0], atol=1e-15)
    doc = {"name": "slider", "links": [{"name": "base"}, {"name": "car", "parent_joint": "j",
                                                          "origin": {"xyz": [0, 0.1, 0]}}],
           "joints": [{"name": "j", "type": "prismatic", "parent_link": "base",
                       "origin": {"rpy": [0, 0, np.pi / 2]}, "axis": [1, 0, 0],
                       "limits": {"position": [-0.5, 0.5], "velocity": 1, "acceleration": 2}}]}
    m = L.RobotModel.from_dict(doc)
    p = L.forward_kinematics_batch(m, L.ConfigBatch([[0.3]]))
    assert np.allclose(p.translations[0, 1], [-0.1, 0.3, 0], atol=1e-15)
    with pytest.raises(L.LimitViolationError) as err:
        L.forward_kinematics_batch(m, L.ConfigBatch([[0.0], [0.9]]))
    assert (1, 0) in err.value.violations


def test_alignment(L):
    # test_placement.py:55-87
    grid = L.EnvGrid(1.0, 0.1)
    a = L.compute_alignment(np.float64([0.10, 0.05, 0.05]), grid, 0.3)
    assert list(a.anchor) == [8, 7, 7] and np.allclose(a.delta_t, [-0.05, 0, 0], atol=1e-15)
    a = L.compute_alignment(np.float64([1.05, 0.0, 0.0]), grid, 0.3)
    assert list(a.anchor) == [17, 7, 7]
    with pytest.raises(L.NoOverlapError):
        L.compute_alignment(np.float64([1.7, 0.0, 0.0]), grid, 0.3)
    rng = np.random.default_rng(5)
    t = rng.uniform(-0.99, 0.99, size=(100_000, 3))
    a = L.compute_alignment(t, grid, 0.3)
    from oracle import linksdf_oracle as O

    ra, rd, _ = O.align(t, O.Env(1.0, 0.1), 0.3)
    assert np.array_equal(a.anchor, ra) and np.array_equal(a.delta_t, rd)


# ----------------------------------------------------------------------------- obstacles


@pytest.mark.parametrize("name", ["scene_c1", "scene_c2", "scene_small", "scene_arm7"])
def test_voxelize(L, name):
    g = golden(name)
    grid = L.EnvGrid(float(g["env_extent"]), float(g["env_res"]))
    v = L.voxelize_pointcloud(g["points"], grid)
    assert np.array_equal(v.indices, g["indices"])
    assert v.n_dropped == int(g["n_dropped"]) and v.n_points == int(g["n_points"])
    v32 = L.voxelize_pointcloud(g["points"].astype(np.float32), grid)
    from oracle import linksdf_oracle as O

    idx, _, drop = O.voxelize(g["points"].astype(np.float32), O.Env(float(g["env_extent"]), float(g["env_res"])))
    assert np.array_equal(v32.indices, idx) and v32.n_dropped == drop


def test_voxelize_edges(L):
    # test_query.py:105-136 + face/NaN/empty cases
    grid = L.EnvGrid(1.0, 0.1)
    v = L.voxelize_pointcloud(np.empty((0, 3)), grid)
    assert v.n_occupied == 0 and v.n_points == 0 and v.n_dropped == 0
    v = L.voxelize_pointcloud(np.tile(np.float64([0.31, 0.02, -0.44]), (1000, 1)), grid)
    assert v.n_occupied == 1 and v.n_points == 1000
    v = L.voxelize_pointcloud(np.float64([[0, 0, 0], [2, 0, 0], [0, -3, 0], [1.0, 0, 0], [-1.0, 0, 0],
                                          [np.nan, 0, 0]]), grid)
    assert v.n_dropped == 4 and v.indices.tolist() == [[0, 10, 10], [10, 10, 10]]
    assert np.array_equal(L.voxel_index_of(np.float64([0.05, 0.05, 0.05]), grid), [10, 10, 10])
    with pytest.raises(L.OutOfBoundsError):
        L.voxel_index_of(np.float64([1.0, 0.0, 0.0]), grid)


# ----------------------------------------------------------------------------- stage 2a


def test_build_primitives_bit_exact(L):
    b = golden("builds")
    from tests.test_hostcheck import _prim_params  # noqa: F401  (same parameter mapping)

    for key in [k for k in b.files if k.startswith("prim_") and not k.endswith("_json")]:
        geom = json.loads(bytes(b[key + "_json"]).decode())
        shape = {"sphere": lambda g: L.Sphere(g["radius"], center=g.get("center", (0, 0, 0))),
                 "capsule": lambda g: L.Capsule(g["radius"], g["half_length"], axis=g.get("axis", (0, 0, 1))),
                 "box": lambda g: L.Box(g["half_extents"])}[geom["type"]](geom)
        s = L.build_link_sdf(shape, 0.2, 0.01)
        assert np.array_equal(s.values, b[key]), key


def test_build_meshes(L):
    b = golden("builds")
    for name in ("ico", "box", "tiltbox", "open"):
        m = L.TriangleMesh(b[f"mesh_{name}_V"], b[f"mesh_{name}_F"])
        e, r = b[f"mesh_{name}_er"]
        s = L.build_link_sdf(m, e, r)
        ref = b[f"mesh_{name}"]
        assert np.abs(s.values - ref).max() <= MESH_TOL, name
        assert np.mean(s.values == ref) > 0.999, name


def test_mesh_culling_is_exact(L):
    """The culled build (compact cell blocks: nearest-tile-first box culling
    of the distance and of the ray-parity tests) == the same tests on the
    cell centres in a random order (CTA boxes span the domain: almost
    nothing culled), bit for bit, signed and open meshes."""
    rng = np.random.default_rng(5)
    ico = L.make_icosphere(0.08, subdivisions=3)
    shifted = L.TriangleMesh(ico.vertices + np.float64([0.03, -0.02, 0.05]), ico.triangles)
    opened = L.TriangleMesh(ico.vertices, ico.triangles[:-40])
    for mesh, signed in ((shifted, True), (L.make_box_mesh([0.05, 0.03, 0.07]), True), (opened, False)):
        sdf = L.build_link_sdf(mesh, 0.16, 0.01)
        ax = [sdf.cell_centers_1d(a) for a in range(3)]
        X, Y, Z = np.meshgrid(*ax, indexing="ij")
        pts = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)
        perm = rng.permutation(len(pts))
        d = np.empty(len(pts))
        d[perm] = L.exact_point_distance(mesh, pts[perm], signed=signed)
        assert np.array_equal(np.asarray(sdf.values).reshape(-1), d.astype(np.float32))


def test_scene_grids_bit_exact(L):
    g = golden("scene_c1")
    _, _, sdfs, _ = _scene(L, g)
    for k, s in enumerate(sdfs):
        assert np.array_equal(s.values, g["grids"][k])
    g2 = golden("scene_c2")
    _, _, sdfs2, _ = _scene(L, g2)
    cells = g2["grid_cells"]
    for k, s in enumerate(sdfs2):
        v = s.values
        assert np.array_equal(v[cells[:, 0], cells[:, 1], cells[:, 2]], g2["grid_samples"][k])
        assert v.astype(np.float64).sum() == g2["grid_sums"][k]


def test_trilinear(L):
    t = golden("trilinear")
    s = L.LinkSdf(float(t["extent"]), float(t["res"]), t["values"], 0)
    assert np.array_equal(L.trilinear_sample(s, t["pts"]), t["out"])


# ----------------------------------------------------------------------------- placement / assembly


def test_place_and_assemble_bit_exact(L):
    g = golden("scene_small")
    robot, grid, sdfs, window = _scene(L, g)
    gl = g["geometry_links"]
    poses = L.LinkPoseBatch(rotations=g["R"][:, gl], translations=g["T"][:, gl])
    prov = L.ExactTransformProvider(window)
    fields = list(L.place_links_batch(sdfs, poses, grid, prov))
    for c, li, f in fields:
        assert np.array_equal(f.anchor, g["anchors"][c, li])
        assert np.array_equal(f.values, g["windows"][c, li])
    batch = L.assemble_robot_sdfs(((c, f) for c, _, f in fields), grid, len(g["q"]), float(g["d_far_global"]))
    assert np.array_equal(batch.values, g["batch"])
    obs = L.voxelize_pointcloud(g["points"], grid)
    d, link, voxel = L.query_min_distances(batch, obs, return_argmin=True)
    assert np.array_equal(d, g["d"]) and np.array_equal(voxel, g["voxel"])
    pl = L.per_link_min_distances(iter(fields), obs, len(g["q"]), len(gl), float(g["d_far_global"]))
    assert np.array_equal(pl, g["per_link"])
    traj = L.TrajectorySdf.from_poses(sdfs, poses, grid, prov)
    assert np.array_equal(traj.values, g["batch"])


# ----------------------------------------------------------------------------- stages 3+4


@pytest.mark.parametrize("name", ["scene_c1", "scene_c2", "scene_small", "scene_arm7"])
def test_direct_query_stage_isolated(L, name):
    """Reference poses in, (d, link, voxel) out: bit-exact against the reference."""
    g = golden(name)
    robot, grid, sdfs, window = _scene(L, g)
    gl = g["geometry_links"]
    poses = L.LinkPoseBatch(rotations=g["R"][:, gl], translations=g["T"][:, gl])
    traj = L.TrajectorySdf.from_poses(sdfs, poses, grid, L.ExactTransformProvider(window))
    obs = L.voxelize_pointcloud(g["points"], grid)
    (d, link, voxel), stats = L.query_min_distances(traj, obs, return_stats=True, return_argmin=True)
    assert stats["gathers"] == len(g["q"]) * len(g["indices"])
    assert np.array_equal(d, g["d"])
    assert np.array_equal(link, g["link"])
    assert np.array_equal(voxel, g["voxel"])
    assert np.array_equal(traj.per_link_min_distances(obs), g["per_link"])


def test_grids_pinned_in_l2(L):
    """The packed grids live in one arena marked persisting in L2; results equal the unpinned query's."""
    g = golden("scene_c2")
    robot, grid, sdfs, window = _scene(L, g)
    gl = g["geometry_links"]
    poses = L.LinkPoseBatch(rotations=g["R"][:, gl], translations=g["T"][:, gl])
    traj = L.TrajectorySdf.from_poses(sdfs, poses, grid, L.ExactTransformProvider(window))
    assert traj.l2_pinned_bytes > 0
    base = traj._arena.data_ptr()
    sizes = [s.packed_values().numel() * 4 for s in sdfs]
    assert [traj._table[i].packed_dev for i in range(len(sdfs))] == [base + sum(sizes[:i]) for i in range(len(sdfs))]
    plain = L.TrajectorySdf(sdfs, grid, window, traj.R, traj.dt, traj.anchor, pin_l2=False)
    obs = L.voxelize_pointcloud(g["points"], grid)
    a = L.query_min_distances(traj, obs, return_argmin=True)
    b = L.query_min_distances(plain, obs, return_argmin=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.array_equal(a[0], g["d"]) and np.array_equal(a[1], g["link"]) and np.array_equal(a[2], g["voxel"])


@pytest.mark.parametrize("name", ["scene_c1", "scene_c2", "scene_arm7"])
def test_full_pipeline_from_configs(L, name):
    g = golden(name)
    robot, grid, sdfs, window = _scene(L, g)
    d, link, voxel = L.query_trajectory(robot, g["q"], sdfs, grid, window, g["points"])
    assert np.abs(d.astype(np.float64) - g["d"]).max() <= D_TOL
    assert np.array_equal(link, g["link"]) and np.array_equal(voxel, g["voxel"])


def test_checker_graph_path(L):
    g = golden("scene_c2")
    robot, grid, sdfs, window = _scene(L, g)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(len(g["q"]), 40_000, np.float64)
    for _ in range(3):  # replay determinism
        d, link, voxel = chk.query(g["q"], g["points"])
        assert np.abs(d.astype(np.float64) - g["d"]).max() <= D_TOL
        assert np.array_equal(link, g["link"]) and np.array_equal(voxel, g["voxel"])
    q_bad = g["q"].copy()
    q_bad[3, 1] = 9.0
    with pytest.raises(L.LimitViolationError) as err:
        chk.query(q_bad, g["points"])
    assert (3, 1) in err.value.violations


@pytest.mark.parametrize("depth", [2, 3])
def test_checker_pipeline(L, depth):
    """CheckerPipeline (cycles in flight, copy-engine transfers) == one-at-a-time checker, cycle by cycle."""
    from paper_2309_12543_b200 import scenarios as S

    g = golden("scene_c2")
    robot, grid, sdfs, window = _scene(L, g)
    C = len(g["q"])
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(C, 40_000, np.float32)
    pipe = L.CheckerPipeline(robot, sdfs, grid, window, C, 40_000, np.float32, depth=depth)
    cycles = [(S.random_configs(_doc(g), C, seed=k), S.human_cloud(30_000 + 1000 * k, seed=k).astype(np.float32))
              for k in range(7)]
    want = [chk.query(q, p) for q, p in cycles]
    tickets = [pipe.submit(q, p) for q, p in cycles[:depth]]
    got = []
    for k in range(len(cycles)):
        got.append(pipe.result(tickets[k]))
        if k + depth < len(cycles):
            tickets.append(pipe.submit(*cycles[k + depth]))
    for (d0, l0, v0), (d1, l1, v1) in zip(want, got):
        assert np.array_equal(d0, d1) and np.array_equal(l0, l1) and np.array_equal(v0, v1)
    q_bad = cycles[0][0].copy()
    q_bad[5, 2] = 9.0
    with pytest.raises(L.LimitViolationError):
        pipe.result(pipe.submit(q_bad, cycles[0][1]))
    # a bad cycle whose slot is recycled before its result() call: the later
    # submissions go through, its own result() raises, the others return
    bad = pipe.submit(q_bad, cycles[0][1])
    later = [pipe.submit(q, p) for q, p in cycles[1:1 + depth]]
    for k, t in enumerate(later):
        d1, l1, v1 = pipe.result(t)
        assert np.array_equal(d1, want[k + 1][0]) and np.array_equal(l1, want[k + 1][1])
    with pytest.raises(L.LimitViolationError):
        pipe.result(bad)


def test_known_answer_tie_clamp_empty(L):
    k = golden("known_answer")
    grid = L.EnvGrid(1.0, 0.1)
    sdfs = [L.build_link_sdf(L.Sphere(0.12), 0.3, 0.01, link_id=0),
            L.build_link_sdf(L.Box([0.05, 0.05, 0.05]), 0.3, 0.01, link_id=1)]
    for s, ref in zip(sdfs, k["grids"]):
        assert np.array_equal(s.values, ref)
    window = L.WindowGeometry.build(0.3, grid)
    traj = L.TrajectorySdf.from_poses(sdfs, L.LinkPoseBatch(k["R"], k["T"]), grid, L.ExactTransformProvider(window))
    for name in ("tie", "far", "empty"):
        idx = k[f"{name}_indices"]
        obs = L.ObstacleVoxelSet(indices=idx, grid=grid, n_points=len(idx), n_dropped=0)
        d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
        assert np.array_equal(d, k[f"{name}_d"]), name
        assert np.array_equal(link, k[f"{name}_link"]), name
        assert np.array_equal(voxel, k[f"{name}_voxel"]), name


def test_unsorted_and_duplicate_obstacles(L):
    """General index lists: first-occurrence argmin like numpy (query.py:146)."""
    from oracle import linksdf_oracle as O

    g = golden("scene_small")
    robot, grid, sdfs, window = _scene(L, g)
    gl = g["geometry_links"]
    poses = L.LinkPoseBatch(rotations=g["R"][:, gl], translations=g["T"][:, gl])
    traj = L.TrajectorySdf.from_poses(sdfs, poses, grid, L.ExactTransformProvider(window))
    rng = np.random.default_rng(3)
    idx = g["indices"][rng.permutation(len(g["indices"]))]
    idx = np.concatenate([idx, idx[:50]])
    obs = L.ObstacleVoxelSet(indices=idx, grid=grid, n_points=len(idx), n_dropped=0)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    env = O.Env(float(g["env_extent"]), float(g["env_res"]))
    anchors = g["anchors"]
    rd, rl, rv = O.argmin_oracle(g["batch"], g["windows"], anchors, idx, float(g["d_far_global"]))
    assert np.array_equal(d, rd) and np.array_equal(link, rl) and np.array_equal(voxel, rv)
    assert env.dims[0] == grid.dims[0]


def test_stream_min_distances(L):
    g = golden("scene_small")
    robot, grid, sdfs, window = _scene(L, g)
    traj = L.TrajectorySdf.from_configs(robot, g["q"], sdfs, grid, window)
    frames = [(float(i), g["points"]) for i in range(3)] + [(3.0, np.empty((0, 3)))]
    rows = list(L.stream_min_distances(traj, frames))
    assert all(np.array_equal(r[1], rows[0][1]) for r in rows[:3])
    assert np.abs(rows[0][1].astype(np.float64) - g["d"]).max() <= D_TOL  # the reference's query (query.py:294-306)
    assert [r[0] for r in rows] == [0.0, 1.0, 2.0, 3.0]
    assert np.all(rows[3][1] == np.float32(traj.d_far_global))


# ----------------------------------------------------------------------------- stage 2b


def test_mlp_predict(L):
    m = golden("mlp")
    model = L.TinyMlp(m["w1"], m["b1"], m["w2"], m["b2"])
    y = model.predict(m["R"])
    assert np.abs(y - m["predict"]).max() <= MLP_TOL
    g = L.infer_grid_transform(model, m["R"], m["dt"], 0.3)
    assert np.abs(g - m["infer"]).max() <= MLP_TOL
    ex = L.grid_transform_exact(m["R"], m["dt"], 0.3, m["masked_points"])
    assert np.array_equal(ex, m["exact"])


@pytest.mark.parametrize("tc,fused", [(False, False), (True, False), (True, True)])
def test_neural_placement(L, tc, fused):
    """place_links_batch with NeuralTransformProvider, fully on the device
    (TinyMlp on tensor cores or CUDA cores -> provider-coordinate sampler, or
    the fused MLP + sampler kernel), vs
    the oracle's numpy MLP transform + trilinear (approx.py:292-306,
    placement.py:300-313): window values within 1e-5 m."""
    from oracle import linksdf_oracle as O

    g, m = golden("scene_small"), golden("mlp")
    robot, grid, sdfs, window = _scene(L, g)
    model = L.TinyMlp(m["w1"], m["b1"], m["w2"], m["b2"])
    prov = L.NeuralTransformProvider(model, window, use_tensor_cores=tc, fused=fused)
    assert prov.fused == fused
    gl = [int(i) for i in g["geometry_links"]]
    R, T = g["R"][:, gl], g["T"][:, gl]
    fields = list(L.place_links_batch(sdfs, L.LinkPoseBatch(rotations=R, translations=T), grid, prov))
    e_r, r_r = float(g["e_r"]), float(g["r_r"])
    env = O.Env(float(g["env_extent"]), float(g["env_res"]))
    _, dt, _ = O.align(T.reshape(-1, 3), env, e_r)
    dt = dt.reshape(T.shape)
    keep = O.window_mask(e_r, env).ravel(order="F")
    worst = 0.0
    for c, li, f in fields:
        G = O.mlp_transform(m["w1"], m["b1"], m["w2"], m["b2"], R[c, li], dt[c, li], e_r)
        s = O.trilinear(sdfs[li].values, e_r, r_r, (G * e_r).reshape(-1, 3))
        vals = f.values.ravel(order="F")
        assert np.all(vals[~keep] == np.float32(sdfs[li].d_far))
        worst = max(worst, float(np.abs(vals[keep].astype(np.float64) - s).max()))
    assert worst <= 1e-5, worst


def test_sphere_baseline(L):
    from oracle import linksdf_oracle as O

    g = golden("scene_small")
    robot = L.RobotModel.from_dict(_doc(g))
    grid = L.EnvGrid(float(g["env_extent"]), float(g["env_res"]))
    li = np.int64([1, 2, 3, 6])
    centers = np.float64([[0, 0, 0.02], [0, 0, -0.03], [0.01, 0, 0], [0, 0, 0]])
    radii = np.float64([0.08, 0.07, 0.06, 0.05])
    sph = L.SphereRobotModel(li, centers, radii)
    poses = L.LinkPoseBatch(g["R"], g["T"])
    obs = L.voxelize_pointcloud(g["points"], grid)
    d, st = L.sphere_baseline_distances(sph, poses, obs, grid, return_stats=True)
    assert st["distance_evals"] == len(g["q"]) * 4 * obs.n_occupied
    tgt = O.Env(float(g["env_extent"]), float(g["env_res"])).centers(obs.indices)
    world = np.einsum("bsij,sj->bsi", g["R"][:, li], centers) + g["T"][:, li]
    ref = (np.linalg.norm(world[:, :, None] - tgt[None, None], axis=-1) - radii[None, :, None]).min(axis=(1, 2))
    assert np.abs(d - ref).max() <= 1e-12
    assert robot.n_links == 7


# ----------------------------------------------------------------------------- full-size properties


def test_config2_full_size_properties(L):
    """BASELINE config 2 at full size: direct == dense gather, oracle on a subset, invariances."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG2
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=0)
    pts = S.cloud_for(shape, seed=0)
    traj = L.TrajectorySdf.from_configs(robot, q, sdfs, grid, window)
    obs = L.voxelize_pointcloud(pts, grid)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    dense = L.RobotSdfBatch(traj.device_values(), grid, traj.d_far_global)
    d2, _, v2 = L.query_min_distances(dense, obs, return_argmin=True)
    assert np.array_equal(d, d2) and np.array_equal(voxel, v2)
    # oracle (reference restatement) on 12 waypoints of the full cloud
    sub = np.arange(0, shape.n_waypoints, 42)
    grids = [s.values for s in sdfs]
    rd, rl, rv = O.run_pipeline(shape.robot, q[sub], pts, shape.grid_extent, shape.grid_res,
                                shape.link_extent, grids, [shape.link_res] * len(grids))
    assert np.abs(d[sub].astype(np.float64) - rd).max() <= D_TOL
    assert np.array_equal(link[sub], rl) and np.array_equal(voxel[sub], rv)
    # permutation of the cloud changes nothing; a superset never increases d
    perm = np.random.default_rng(1).permutation(len(pts))
    dp = L.query_min_distances(traj, L.voxelize_pointcloud(pts[perm], grid))
    assert np.array_equal(dp, d)
    more = np.concatenate([pts, S.human_cloud(20_000, seed=9)])
    dm = L.query_min_distances(traj, L.voxelize_pointcloud(more, grid))
    assert np.all(dm <= d)
    # waypoint sharding (the multi-GPU partition) is exact: shards == whole
    halves = [L.TrajectorySdf.from_configs(robot, q[s], sdfs, grid, window)
              for s in (slice(0, 250), slice(250, 500))]
    ds = np.concatenate([L.query_min_distances(h, obs) for h in halves])
    assert np.array_equal(ds, d)


def test_config4_shape_large_batch(L):
    """Config-4 shape (arm7g, crowd, 64^3), 8,000 waypoints: the whole batch ==
    the same waypoints in chunks (dynamic task fetch and grab sizes differ) ==
    the oracle on a subset; the graph checker agrees bit for bit."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG4
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    C = 8000  # >= the FK thread-per-configuration threshold; the 2,000 chunks use the 3-phase kernel
    q = S.random_configs(shape.robot, C, seed=3)
    pts = S.cloud_for(shape, seed=3)[:300_000].astype(np.float32)
    obs = L.voxelize_pointcloud(pts, grid)
    traj = L.TrajectorySdf.from_configs(robot, q, sdfs, grid, window)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    parts = [L.query_min_distances(L.TrajectorySdf.from_configs(robot, q[a:a + 2000], sdfs, grid, window), obs,
                                   return_argmin=True) for a in range(0, C, 2000)]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), d)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), link)
    assert np.array_equal(np.concatenate([p[2] for p in parts]), voxel)
    sub = np.arange(0, C, 1000)
    grids = [s.values for s in sdfs]
    rd, rl, rv = O.run_pipeline(shape.robot, q[sub], pts, shape.grid_extent, shape.grid_res,
                                shape.link_extent, grids, [shape.link_res] * len(grids))
    assert np.abs(d[sub].astype(np.float64) - rd).max() <= D_TOL
    assert np.array_equal(link[sub], rl) and np.array_equal(voxel[sub], rv)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(C, len(pts), np.float32)
    assert chk.link_major  # large batches keep the poses link-major
    for _ in range(2):
        dc, lc, vc = chk.query(q, pts)
        assert np.array_equal(dc, d) and np.array_equal(lc, link) and np.array_equal(vc, voxel)
    # the link-major poses (lsdf_fk_align_link_major) == the configuration-major ones, bit for bit
    for a, b in zip(chk.traj.config_major(), (traj.R, traj.dt, traj.anchor)):
        assert np.array_equal(a.reshape(C, len(sdfs), -1).cpu().numpy(), b.reshape(C, len(sdfs), -1).cpu().numpy())
    # the scan orders the links by the previous cycle's argmin counts (kept in
    # the query workspace); any order must give the same answer: force some
    a256 = lambda n: (n + 255) // 256 * 256  # noqa: E731
    G = len(sdfs)
    import torch

    hist = chk.qws[a256(C * 4) + a256(C * 8) + a256(C * G * 4):][: 4 * G].view(torch.int32)
    assert int(hist.sum().item()) == int((link >= 0).sum())  # the last cycle's argmin counts
    for counts in (np.arange(G)[::-1], np.arange(G), np.roll(np.arange(G), 3), np.zeros(G)):
        hist.copy_(torch.from_numpy(counts.astype(np.int32) * 100))
        dc, lc, vc = chk.query(q, pts)
        assert np.array_equal(dc, d) and np.array_equal(lc, link) and np.array_equal(vc, voxel)


@pytest.mark.parametrize("seed,cloud", [(0, "uniform"), (1, "uniform"), (2, "clusters"), (3, "clusters")])
def test_direct_equals_dense_on_adversarial_grids(L, seed, cloud):
    """Random (non-Lipschitz) grid values, random rotations, a dense cloud or a
    few tight clusters (most windows empty: the brick box test skips them):
    the screened direct kernel must select exactly what the dense gather selects."""
    rng = np.random.default_rng(seed)
    grid = L.EnvGrid(1.0, 0.05)
    e_r = 0.3
    window = L.WindowGeometry.build(e_r, grid)
    sdfs = []
    for li in range(3):
        vals = rng.normal(0.0, 0.2, size=(30, 30, 30)).astype(np.float32)
        if li == 1:
            vals = np.round(vals * 8) / 8  # many exact ties
        sdfs.append(L.LinkSdf(e_r, 0.02, vals, li))
    C = 40
    R = L.sample_rotations(rng, C * 3).reshape(C, 3, 3, 3)
    T = rng.uniform(-0.6, 0.6, size=(C, 3, 3))
    traj = L.TrajectorySdf.from_poses(sdfs, L.LinkPoseBatch(R, T), grid, L.ExactTransformProvider(window))
    if cloud == "uniform":
        pts = rng.uniform(-1, 1, size=(20_000, 3))
    else:  # tight blobs, one on a brick boundary and one in a grid corner
        centres = np.array([[0.2, -0.2, 0.2], [-0.8, 0.8, -0.8], [0.0, 0.0, 0.0], [0.95, 0.95, 0.95]])
        pts = np.concatenate([c + rng.normal(0, 0.03, size=(100, 3)) for c in centres])
    obs = L.voxelize_pointcloud(pts, grid)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    dense = L.RobotSdfBatch(traj.device_values(), grid, traj.d_far_global)
    d2, _, v2 = L.query_min_distances(dense, obs, return_argmin=True)
    assert np.array_equal(d, d2) and np.array_equal(voxel, v2)
    # link: lowest link whose window value at the winning voxel equals d
    fields = list(L.place_links_batch(sdfs, L.LinkPoseBatch(R, T), grid, L.ExactTransformProvider(window)))
    pl = L.per_link_min_distances(iter(fields), obs, C, 3, traj.d_far_global)
    assert np.array_equal(traj.per_link_min_distances(obs), pl)
    for c in range(C):
        if link[c] >= 0:
            assert pl[c, link[c]] == d[c]
            assert np.all(pl[c, : link[c]] > d[c]) or voxel[c] >= 0


@pytest.mark.parametrize("cloud", ["dense", "sparse"])
def test_segment_bound_exact_on_noisy_grids(L, cloud):
    """Throughput-sized batch (segment bound active) on capsule-like grids
    with noise (the bound's kappas come from the values): direct == dense
    gather, and == the same waypoints in small chunks (bound inactive).
    The sparse cloud leaves a few occupied cells per window, many in the outer
    shell past the link grid's cell-centre hull (sample = far value, above
    the segment's upper bound): the threshold must not be lowered there."""
    rng = np.random.default_rng(11)
    grid = L.EnvGrid(1.0, 0.05)
    e_r, r_r = 0.3, 0.02
    window = L.WindowGeometry.build(e_r, grid)
    ax = -e_r + (np.arange(30) + 0.5) * r_r
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    sdfs = []
    for li, (r, hl) in enumerate(((0.06, 0.08), (0.04, 0.0), (0.05, 0.05))):
        t = np.clip(Z, -hl, hl)
        v = np.sqrt(X * X + Y * Y + (Z - t) ** 2) - r + rng.normal(0.0, 0.004, size=X.shape)
        if li == 2:
            v = np.round(v * 64) / 64  # exact ties
        sdfs.append(L.LinkSdf(e_r, r_r, v.astype(np.float32), li))
    C = 13_000  # 39,000 tasks: above the segment-bound threshold
    R = L.sample_rotations(rng, C * 3).reshape(C, 3, 3, 3)
    T = rng.uniform(-0.6, 0.6, size=(C, 3, 3))
    poses = L.LinkPoseBatch(R, T)
    prov = L.ExactTransformProvider(window)
    traj = L.TrajectorySdf.from_poses(sdfs, poses, grid, prov)
    obs = L.voxelize_pointcloud(rng.uniform(-1, 1, size=(20_000 if cloud == "dense" else 400, 3)), grid)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    dense = L.RobotSdfBatch(traj.device_values(), grid, traj.d_far_global)
    d2, _, v2 = L.query_min_distances(dense, obs, return_argmin=True)
    assert np.array_equal(d, d2) and np.array_equal(voxel, v2)
    if cloud == "sparse":
        assert np.mean(link >= 0) > 0.3  # most waypoints see an obstacle: the case is exercised
    for a in range(0, C, 2600):
        part = L.TrajectorySdf.from_poses(sdfs, L.LinkPoseBatch(R[a:a + 2600], T[a:a + 2600]), grid, prov)
        dc, lc, vc = L.query_min_distances(part, obs, return_argmin=True)
        assert np.array_equal(dc, d[a:a + 2600]) and np.array_equal(lc, link[a:a + 2600])
        assert np.array_equal(vc, voxel[a:a + 2600])


def _hull_trap_scenes(n_scenes, seed=0):
    """Poses where the shell scan's segment bound meets a window cell outside
    the link grid's cell-centre hull (sample = far value, above the segment's
    upper bound) BEFORE an in-hull cell holding the true minimum, which the
    unguarded threshold update would then skip.  CPU search with
    the oracle's trilinear; returns the link grid and, per scene, (R, dt, cells)."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200.placement import _axis_offsets

    import paper_2309_12543_b200 as L

    rng = np.random.default_rng(seed)
    e_r, r_r = 0.3, 0.02
    ax = -e_r + (np.arange(30) + 0.5) * r_r
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    vals = (np.sqrt(X * X + Y * Y + (Z - np.clip(Z, -0.2, 0.2)) ** 2) - 0.02).astype(np.float32)  # long thin capsule
    sdf = L.LinkSdf(e_r, r_r, vals, 0)
    a, u, length, k_lo, k_hi = sdf.segment_bound()
    a, u = np.asarray(a), np.asarray(u)
    core = sdf.core_radius()
    grid = L.EnvGrid(1.0, 0.05)
    w = L.WindowGeometry.build(e_r, grid)
    h = w.host_tables()
    off = _axis_offsets(w.extent, w.grid, False)
    cells = h["shell_cells"][: w.n_masked].astype(np.int64)
    m = np.stack([cells & 0xFF, (cells >> 8) & 0xFF, (cells >> 16) & 0xFF], 1)
    Pm = np.stack([off[0][m[:, 0]], off[1][m[:, 1]], off[2][m[:, 2]]], 1)
    rad = h["shell_radius"][: w.n_masked]
    hull, clamp = e_r - r_r / 2, np.float32(e_r)
    chunk = np.arange(len(Pm)) // 32
    scenes = []
    while len(scenes) < n_scenes:
        R = L.sample_rotations(rng, 1)[0]
        dt = rng.uniform(-0.024, 0.024, 3)
        p = (Pm - dt) @ R
        v = O.trilinear(vals, e_r, r_r, p).astype(np.float64)
        tt = np.clip((p - a) @ u, 0, length)
        d = np.linalg.norm(p - a - tt[:, None] * u, axis=1)
        outside = np.any(np.abs(p) > hull + 1e-3, axis=1)
        for o in np.nonzero(outside)[0]:
            th = min(clamp, d[o] + k_hi)
            skipped = (d - k_lo > th) | (rad[chunk * 32] - (np.linalg.norm(dt) + core) > th)
            cand = np.nonzero((chunk > chunk[o]) & ~outside & skipped & (v < clamp - 0.01))[0]
            if d[o] - k_lo <= clamp and len(cand):
                scenes.append((R, dt, m[o], m[cand[0]]))
                break
    return sdf, grid, w, scenes


def test_segment_bound_guard_outside_hull(L):
    """Throughput-sized batch whose windows hold exactly two occupied cells: one
    past the link grid's cell-centre hull in an early shell chunk, one inside
    it farther out with the true minimum.  The direct kernel (segment bound
    on) must equal the dense gather and the same poses as a small batch."""
    sdf, grid, window, scenes = _hull_trap_scenes(27)
    W = int(window.dims[0])
    env_c = lambda j: -1.0 + (np.asarray(j) + 0.5) * 0.05  # noqa: E731  voxel centres
    Rs, Ts, pts = [], [], []
    for k, (R, dt, co, ci) in enumerate(scenes):  # 27 disjoint windows on a 3 x 3 x 3 lattice of anchors
        anchor = 13 * np.array([k % 3, (k // 3) % 3, k // 9])
        Rs.append(R)
        Ts.append(env_c(anchor + W // 2) + dt)
        pts += [env_c(anchor + co), env_c(anchor + ci)]
    Rs, Ts = np.asarray(Rs), np.asarray(Ts)
    obs = L.voxelize_pointcloud(np.asarray(pts), grid)
    assert obs.n_occupied == 2 * len(scenes)
    prov = L.ExactTransformProvider(window)
    small = L.TrajectorySdf.from_poses([sdf], L.LinkPoseBatch(Rs[:, None], Ts[:, None]), grid, prov)
    d0, l0, v0 = L.query_min_distances(small, obs, return_argmin=True)
    dense = L.RobotSdfBatch(small.device_values(), grid, small.d_far_global)
    d1, _, v1 = L.query_min_distances(dense, obs, return_argmin=True)
    assert np.array_equal(d0, d1) and np.array_equal(v0, v1)
    assert np.all(l0 == 0) and np.all(d0 < np.float32(0.3))  # every trap has its in-hull minimum
    reps = 40_000 // len(scenes) + 1  # > 37,888 tasks: the segment bound is on
    big = L.TrajectorySdf.from_poses([sdf], L.LinkPoseBatch(np.tile(Rs, (reps, 1, 1))[:, None],
                                                            np.tile(Ts, (reps, 1))[:, None]), grid, prov)
    d, link, voxel = L.query_min_distances(big, obs, return_argmin=True)
    assert np.array_equal(d, np.tile(d0, reps)) and np.array_equal(link, np.tile(l0, reps))
    assert np.array_equal(voxel, np.tile(v0, reps))


def test_mlp_tensor_cores(L):
    """tcgen05 kind::tf32 (3xTF32) layer 2 vs the reference prediction and the CUDA-core kernel."""
    import torch

    m = golden("mlp")
    model = L.TinyMlp(m["w1"], m["b1"], m["w2"], m["b2"])
    R = torch.from_numpy(np.ascontiguousarray(m["R"].reshape(-1, 9))).cuda()
    y_tc = model.predict_device(R, use_tensor_cores=True).cpu().numpy().reshape(m["predict"].shape)
    assert np.abs(y_tc - m["predict"]).max() <= MLP_TOL
    rng = np.random.default_rng(4)
    big = L.TinyMlp.random(2103, hidden=32, seed=3)   # the W = 16 window of configs 1-2
    Rb = torch.from_numpy(L.sample_rotations(rng, 300).reshape(-1, 9)).cuda()
    a = big.predict_device(Rb, use_tensor_cores=True).cpu().numpy()
    b = big.predict_device(Rb, use_tensor_cores=False).cpu().numpy()
    scale = np.abs(b).max()
    assert np.abs(a - b).max() <= 1e-6 * max(1.0, scale) * 8
    # new weights (same buffer shapes, possibly the same addresses): the packed copy follows
    big.w2 = np.random.default_rng(9).normal(0, 0.3, size=big.w2.shape).astype(np.float32)
    big._dev = None
    a2 = big.predict_device(Rb, use_tensor_cores=True).cpu().numpy()
    b2 = big.predict_device(Rb, use_tensor_cores=False).cpu().numpy()
    assert np.abs(a2 - b2).max() <= 1e-6 * max(1.0, np.abs(b2).max()) * 8
    # row stride: packed, padded (the default allocation) and odd strides agree bit for bit;
    # 300 rotations = one full and one partial 256-rotation tile
    n = 3 * 2103
    for tc in (True, False):
        ref = big.predict_device(Rb, use_tensor_cores=tc, out=torch.empty((300, n), device="cuda"))
        for ld in (n + 1, n + 27, 6336):
            buf = torch.full((300, ld), 7.0, device="cuda")
            y = big.predict_device(Rb, use_tensor_cores=tc, out=buf[:, :n])
            assert torch.equal(y, ref) and bool((buf[:, n:] == 7.0).all())


def test_obstacle_shards_recombine_exactly(L):
    """Obstacle sharding: per-shard GPU queries + packed-key min == the full query."""
    from paper_2309_12543_b200 import sharding as Sh

    g = golden("scene_c1")
    robot, grid, sdfs, window = _scene(L, g)
    traj = L.TrajectorySdf.from_configs(robot, g["q"], sdfs, grid, window)
    obs = L.voxelize_pointcloud(g["points"], grid)
    full = L.query_min_distances(traj, obs, return_argmin=True)
    for world in (2, 3):
        keys = []
        for r in range(world):
            lo, hi = Sh.shard_range(obs.n_occupied, r, world)
            part = L.ObstacleVoxelSet(indices=obs.indices[lo:hi], grid=grid, n_points=hi - lo, n_dropped=0)
            d, link, voxel = L.query_min_distances(traj, part, return_argmin=True)
            keys.append(Sh.pack_keys(d, link, voxel, traj.n_links, voxel_offset=lo))
        red = np.minimum.reduce([Sh._to_signed(k) for k in keys])
        d, link, voxel = Sh.unpack_keys(Sh._from_signed(red), traj.n_links, traj.d_far_global)
        assert np.array_equal(d, full[0]) and np.array_equal(link, full[1]) and np.array_equal(voxel, full[2])


def test_nccl_sharding_paths_world1(L):
    """The NCCL code paths of sharding.py on one GPU (world size 1): link-sharded
    build == local builds bit for bit; obstacle-sharded query == the full query."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2309_12543_b200 import sharding as Sh

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        g = golden("scene_c1")
        robot, grid, sdfs, window = _scene(L, g)
        geoms = [robot.links[i].geometry for i in robot.geometry_links]
        e_r, r_r = float(g["e_r"]), float(g["r_r"])
        built = Sh.build_link_sdfs_sharded(geoms, e_r, r_r)
        for a, b in zip(built, sdfs):
            assert np.array_equal(np.asarray(a.values), np.asarray(b.values))
        traj = L.TrajectorySdf.from_configs(robot, g["q"], built, grid, window)
        obs = L.voxelize_pointcloud(g["points"], grid)
        full = L.query_min_distances(traj, obs, return_argmin=True)
        d, link, voxel = Sh.query_obstacle_sharded(traj, obs)
        assert np.array_equal(d, full[0]) and np.array_equal(link, full[1]) and np.array_equal(voxel, full[2])
    finally:
        dist.destroy_process_group()


def test_training_matches_reference(L):
    """train_approximator on the GPU (same init, rotation stream, L1 + Adam and
    early-stop rule, approx.py:212-289) vs the reference's own run
    (tests/golden/make_training.py): weights within 1e-6 after 300 steps,
    the same checkpoints, errors within 1e-6 relative."""
    g = golden("training")
    cfg = L.TrainingConfig(steps=300, eval_every=100, screen_size=128, val_size=512, target_max_error=1.0, seed=3)
    m = L.train_approximator(g["points"], cfg)
    for k in ("w1", "b1", "w2", "b2"):
        assert np.abs(getattr(m, k) - g[k]).max() <= 1e-6, k
    hist = np.asarray(m.history, dtype=np.float64)
    assert hist.shape == g["history"].shape and np.array_equal(hist[:, 0], g["history"][:, 0])
    assert np.allclose(hist[:, 1:], g["history"][:, 1:], rtol=1e-6, atol=0)
    assert abs(m.validation_max_error - float(g["val_max"])) <= 1e-6 * float(g["val_max"])
    with pytest.raises(L.NotConvergedError):
        L.train_approximator(g["points"], L.TrainingConfig(steps=100, eval_every=100, screen_size=64, val_size=128,
                                                           target_max_error=0.01, seed=3))


def test_unstaged_shell_paths(L):
    """A fine environment grid (100^3: the occupancy bitmap does not fit the
    shared-memory stage) and a wide window (W = 32: 17k kept cells, the shell
    list is read from L2): direct == dense gather bit for bit, and the
    oracle on a subset."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200 import scenarios as S

    doc = S.ARM6G
    robot = L.RobotModel.from_dict(doc)
    grid = L.EnvGrid(1.0, 0.02)
    e_r, r_r = 0.32, 0.02
    sdfs = [L.build_link_sdf(robot.links[i].geometry, e_r, r_r, link_id=i) for i in robot.geometry_links]
    window = L.WindowGeometry.build(e_r, grid)
    assert window.n_masked > 4096
    q = S.random_configs(doc, 64, seed=8)
    pts = S.human_cloud(20_000, seed=8)
    traj = L.TrajectorySdf.from_configs(robot, q, sdfs, grid, window)
    obs = L.voxelize_pointcloud(pts, grid)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    dense = L.RobotSdfBatch(traj.device_values(), grid, traj.d_far_global)
    d2, _, v2 = L.query_min_distances(dense, obs, return_argmin=True)
    assert np.array_equal(d, d2) and np.array_equal(voxel, v2)
    sub = np.arange(0, 64, 8)
    grids = [s.values for s in sdfs]
    rd, rl, rv = O.run_pipeline(doc, q[sub], pts, 1.0, 0.02, e_r, grids, [r_r] * len(grids))
    assert np.abs(d[sub].astype(np.float64) - rd).max() <= D_TOL
    assert np.array_equal(link[sub], rl) and np.array_equal(voxel[sub], rv)


@pytest.mark.parametrize("name", ["scene_c1", "scene_c2", "scene_arm7"])
def test_voxel_major_mode(L, name):
    """The paper's materialized mode, voxel-major: prepare once, then every
    cycle's (d, link, voxel) equal the fused direct query bit for bit (and so
    the reference gather + Appendix-B argmin), over several clouds."""
    from paper_2309_12543_b200 import scenarios as S

    g = golden(name)
    robot, grid, sdfs, window = _scene(L, g)
    traj = L.TrajectorySdf.from_configs(robot, g["q"], sdfs, grid, window)
    dense = traj.materialize()
    assert np.array_equal(dense.values, traj.values)  # the field is the assembled batch
    clouds = [g["points"], S.human_cloud(5000, seed=3), np.zeros((0, 3)), S.crowd_cloud(4, 5000, seed=4)]
    for pts in clouds:
        obs = L.voxelize_pointcloud(pts, grid)
        want = L.query_min_distances(traj, obs, return_argmin=True)
        got = L.query_min_distances(dense, obs, return_argmin=True)
        for a, b in zip(want, got):
            assert np.array_equal(a, b)
    # unsorted list with duplicates: first occurrence in the list
    obs = L.voxelize_pointcloud(g["points"], grid)
    idx = np.concatenate([obs.indices[::-1], obs.indices[:7]])
    part = L.ObstacleVoxelSet(indices=idx, grid=grid, n_points=len(idx), n_dropped=0)
    want = L.query_min_distances(traj, part, return_argmin=True)
    got = L.query_min_distances(dense, part, return_argmin=True)
    for a, b in zip(want, got):
        assert np.array_equal(a, b)


def test_materialized_checker(L):
    """MaterializedChecker (prepare once, graph per cycle) == DistanceChecker, cycle by cycle."""
    from paper_2309_12543_b200 import scenarios as S

    g = golden("scene_c2")
    robot, grid, sdfs, window = _scene(L, g)
    q = g["q"]
    mat = L.MaterializedChecker(robot, sdfs, grid, window, q).prepare(30_000, np.float32)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(len(q), 30_000, np.float32)
    for k, (_, pts) in enumerate(S.moving_human_frames(12, 30_000, seed=2)):
        if k % 3:
            continue
        want = chk.query(q, pts.astype(np.float32))
        got = mat.query(pts.astype(np.float32))
        for a, b in zip(want, got):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("C", [64, 9000])
def test_mixed_link_grids(L, C):
    """Links baked at different resolutions (several launch groups, each with
    its own task counter) and an anisotropic environment grid: direct ==
    dense gather bit for bit, at a latency-sized and a throughput-sized batch."""
    from paper_2309_12543_b200 import scenarios as S

    doc = S.ARM6G
    robot = L.RobotModel.from_dict(doc)
    grid = L.EnvGrid([1.0, 0.8, 0.9], 0.04)
    e_r = 0.32
    res = [0.02, 0.01, 0.02, 0.04, 0.01, 0.02]
    sdfs = [L.build_link_sdf(robot.links[i].geometry, e_r, r, link_id=i) for i, r in zip(robot.geometry_links, res)]
    window = L.WindowGeometry.build(e_r, grid)
    q = S.random_configs(doc, C, seed=12)
    pts = S.human_cloud(30_000, seed=12)
    traj = L.TrajectorySdf.from_configs(robot, q, sdfs, grid, window)
    obs = L.voxelize_pointcloud(pts, grid)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    sub = slice(0, min(C, 2000))
    part = L.TrajectorySdf.from_configs(robot, q[sub], sdfs, grid, window)
    dense = L.RobotSdfBatch(part.device_values(), grid, part.d_far_global)
    d2, _, v2 = L.query_min_distances(dense, obs, return_argmin=True)
    assert np.array_equal(d[sub], d2) and np.array_equal(voxel[sub], v2)
    pl = part.per_link_min_distances(obs)
    for c in range(0, len(d2), 37):
        if link[c] >= 0:
            assert pl[c, link[c]] == d[c] and np.all(pl[c, :link[c]] > d[c])



def _sharded_worker(rank, world, port, out, n_configs=64):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    # gloo: several ranks share the one GPU of this box (a functional check of
    # the exchange; production runs one rank per GPU over NCCL)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S
    from paper_2309_12543_b200.sharding import shard_range

    g = golden("scene_c2")
    robot, grid, sdfs, window = _scene(L, g)
    q = S.random_configs(_doc(g), n_configs, seed=5)
    pts = np.concatenate([S.human_cloud(40_000, seed=5), np.float64([[5.0, 0, 0], [np.nan, 0, 0]])]).astype(np.float32)
    lo, hi = shard_range(len(pts), rank, world)
    ql, qh = shard_range(len(q), rank, world)
    pipe = L.ShardedCloudPipeline(robot, sdfs, grid, window, qh - ql, hi - lo, np.float32, depth=2)
    results = []
    for k in range(3):
        qv, pv = pipe.inputs()
        qv[...] = q[ql:qh]
        pv[...] = pts[lo:hi]
        results.append(pipe.result(pipe.submit()))
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(qh - ql, len(pts), np.float32)
    want = chk.query(q[ql:qh], pts)
    out.put((rank, all(all(np.array_equal(a, b) for a, b in zip(r, want)) for r in results)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_configs", [64, 12_400])
def test_sharded_cloud_pipeline(L, n_configs):
    """Each of 2 ranks uploads half of the cloud; the bitmap all-gather + OR
    merge reproduces one rank voxelizing everything (dropped points too);
    6,200 configurations per rank run the link-major pose path."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q, n_configs)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}


def test_clamp_above_link_far_values(L):
    """d_far_global above the links' own far value (the masked window cells
    then count, query.py:82-83): the full-window kernel path, direct == dense
    gather bit for bit, per-link minima included."""
    g = golden("scene_c1")
    robot, grid, sdfs, window = _scene(L, g)
    clamp = 0.45
    assert all(s.d_far < clamp for s in sdfs)
    traj = L.TrajectorySdf.from_configs(robot, g["q"], sdfs, grid, window, d_far_global=clamp)
    obs = L.voxelize_pointcloud(g["points"], grid)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    dense = L.RobotSdfBatch(traj.device_values(), grid, clamp)
    d2, _, v2 = L.query_min_distances(dense, obs, return_argmin=True)
    assert np.array_equal(d, d2) and np.array_equal(voxel, v2)
    assert np.any(d > max(s.d_far for s in sdfs) - 1e-6) or np.all(d < clamp)
    vm = traj.materialize()
    for a, b in zip(L.query_min_distances(vm, obs, return_argmin=True), (d, link, voxel)):
        assert np.array_equal(a, b)


# ----------------------------------------------------------------------------- plain-C client


@pytest.mark.parametrize("name", ["scene_c2", "scene_arm7"])
def test_c_abi_client(L, name, tmp_path):
    """tests/native/abi_demo.c (C99 + CUDA runtime, no Python in the process) runs FK -> voxelize ->
    fused query through the C ABI; repeated cycles reuse the workspace.  Same answers as the goldens,
    bit-identical to the Python facade."""
    import subprocess

    from paper_2309_12543_b200.build import build_demo
    from tests.native.abi_scene import read_result, write_scene

    g = golden(name)
    robot, grid, sdfs, window = _scene(L, g)
    scene, out = tmp_path / "scene.bin", tmp_path / "out.bin"
    write_scene(scene, robot, sdfs, grid, window, g["q"], g["points"], repeat=3)
    r = subprocess.run([str(build_demo()), str(scene), str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "kernels enqueued" in r.stdout
    d, link, voxel, flags = read_result(out, len(g["q"]))
    assert flags.tolist() == [0, 0]
    assert np.abs(d.astype(np.float64) - g["d"]).max() <= D_TOL
    assert np.array_equal(link, g["link"]) and np.array_equal(voxel, g["voxel"])
    d_py, link_py, voxel_py = L.query_trajectory(robot, g["q"], sdfs, grid, window, g["points"])
    assert np.array_equal(d, d_py) and np.array_equal(link, link_py) and np.array_equal(voxel, voxel_py)


@pytest.mark.parametrize("C", [6161, 6145 + 64])
def test_link_major_checker_ragged_batch(L, C):
    """Link-major poses (lsdf_fk_align_link_major) with a batch that ends inside a
    warp / CTA: the checker == the configuration-major fused query bit for bit."""
    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG4
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    q = S.random_configs(shape.robot, C, seed=9)
    pts = S.cloud_for(shape, seed=9)[:200_000].astype(np.float32)
    traj = L.TrajectorySdf.from_configs(robot, q, sdfs, grid, window)
    ref = L.query_min_distances(traj, L.voxelize_pointcloud(pts, grid), return_argmin=True)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(C, len(pts), np.float32)
    assert chk.link_major
    for _ in range(2):
        got = chk.query(q, pts)
        for a, b in zip(got, ref):
            assert np.array_equal(a, b)
    for a, b in zip(chk.traj.config_major(), (traj.R, traj.dt, traj.anchor)):
        assert np.array_equal(a.reshape(C, len(sdfs), -1).cpu().numpy(), b.reshape(C, len(sdfs), -1).cpu().numpy())
