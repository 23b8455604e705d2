"""GPU parity on the exact inputs bench.py measures (VERDICT r1 "next round" #1).

Fixtures come from the real reference (tests/golden/make_golden_r2.py):
config 2 seeds 21-24 (all 500 waypoints), config 4's seed-11 step (16 of the
65,536 waypoints against the full 1M-point crowd cloud) and the config-3
builds at 128^3.  The full config-4 step is also checked against the dense
gather (the reference's own query on the assembled field) on a 2,000-waypoint
slice, and the W = 128 TinyMlp on tensor cores against the CUDA-core kernel.
Bars as in test_gpu_parity.py: distances from device FK within 1e-6 m,
argmin link / voxel bit-exact, primitive grids bit-exact, meshes 1e-5 m.
"""

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu

D_TOL = 1e-6
MESH_TOL = 1e-5


@pytest.fixture(scope="module")
def L():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_12543_b200 as lib

    return lib


def _digest(a):
    a = np.ascontiguousarray(a)
    return np.float64([a.astype(np.float64).sum(), np.abs(a.astype(np.float64)).sum(), a.size])


def _setup(L, shape):
    robot = L.RobotModel.from_dict(shape.robot)
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    sdfs = [L.build_link_sdf(robot.links[i].geometry, shape.link_extent, shape.link_res, link_id=i)
            for i in robot.geometry_links]
    window = L.WindowGeometry.build(shape.link_extent, grid)
    return robot, grid, sdfs, window


def _device_cycle(chk, q, pts):
    """bench.py's timed path: inputs resident in HBM, one graph replay."""
    import torch

    chk.q_dev.copy_(torch.from_numpy(np.ascontiguousarray(q)))
    chk.p_dev.copy_(torch.from_numpy(np.ascontiguousarray(pts)))
    chk.launch(device_only=True)
    torch.cuda.synchronize()
    return chk.d_dev.cpu().numpy(), chk.link_dev.cpu().numpy(), chk.voxel_dev.cpu().numpy()


def test_config2_bench_seeds_vs_reference(L):
    """Config 2 exactly as benched (seeds 21-24, f32 clouds): the device cycle,
    the host-to-host cycle and the reference agree on every waypoint."""
    from paper_2309_12543_b200 import scenarios as S

    g = golden("bench_c2")
    shape = S.CONFIG2
    robot, grid, sdfs, window = _setup(L, shape)
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(shape.n_waypoints, shape.n_points, np.float32)
    for seed in (21, 22, 23, 24):
        q = S.random_configs(shape.robot, shape.n_waypoints, seed=seed)
        pts = S.cloud_for(shape, seed).astype(np.float32)
        assert np.array_equal(_digest(q), g[f"s{seed}_q_digest"]) and np.array_equal(_digest(pts), g[f"s{seed}_pts_digest"])
        d, link, voxel = _device_cycle(chk, q, pts)
        assert np.abs(d.astype(np.float64) - g[f"s{seed}_d"]).max() <= D_TOL
        assert np.array_equal(link, g[f"s{seed}_link"]) and np.array_equal(voxel, g[f"s{seed}_voxel"])
        assert int(chk.ws[:4].view(__import__("torch").int32).item()) == int(g[f"s{seed}_n_occ"])
        d2, l2, v2 = chk.query(q, pts)
        assert np.array_equal(d2, d) and np.array_equal(l2, link) and np.array_equal(v2, voxel)


def test_config4_bench_step_vs_reference_and_dense(L):
    """Config 4's seed-11 step (65,536 waypoints x 1M points, the bench's
    checker and pipeline): reference on 16 waypoints, the dense gather on a
    2,000-waypoint slice, and the e2e pipeline == the device cycle."""
    import torch

    from paper_2309_12543_b200 import scenarios as S

    g = golden("bench_c4")
    shape = S.CONFIG4
    robot, grid, sdfs, window = _setup(L, shape)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=11)
    pts = S.cloud_for(shape, 11).astype(np.float32)
    assert np.array_equal(_digest(q), g["q_digest"]) and np.array_equal(_digest(pts), g["pts_digest"])
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(shape.n_waypoints, shape.n_points, np.float32)
    d, link, voxel = _device_cycle(chk, q, pts)
    assert int(chk.ws[:4].view(torch.int32).item()) == int(g["n_occ"])
    sub = g["sub"]
    assert np.abs(d[sub].astype(np.float64) - g["d"]).max() <= D_TOL
    assert np.array_equal(link[sub], g["link"]) and np.array_equal(voxel[sub], g["voxel"])
    # the dense gather (the reference's query on the assembled robot SDF) on a slice
    obs = L.voxelize_pointcloud(pts, grid)
    for a in (0, 31_000, shape.n_waypoints - 2000):
        part = L.TrajectorySdf.from_configs(robot, q[a:a + 2000], sdfs, grid, window)
        dense = L.RobotSdfBatch(part.device_values(), grid, part.d_far_global)
        dd, _, vd = L.query_min_distances(dense, obs, return_argmin=True)
        assert np.array_equal(dd, d[a:a + 2000]) and np.array_equal(vd, voxel[a:a + 2000])
        _, lp, _ = L.query_min_distances(part, obs, return_argmin=True)
        assert np.array_equal(lp, link[a:a + 2000])
        del part, dense
    # the e2e throughput path (CheckerPipeline, copy-engine transfers) on the same step
    pipe = L.CheckerPipeline(robot, sdfs, grid, window, shape.n_waypoints, shape.n_points, np.float32, depth=2)
    for _ in range(2):
        qv, pv = pipe.inputs()
        qv[...], pv[...] = q, pts
        dp, lp, vp = pipe.result(pipe.submit())
        assert np.array_equal(dp, d) and np.array_equal(lp, link) and np.array_equal(vp, voxel)


def test_config3_builds_128_vs_reference(L):
    """Config 3 (i) at size: six primitives bit-exact on strided cells (and the
    full-grid sums), the 1,280-triangle icosphere within 1e-5 m."""
    from paper_2309_12543_b200 import scenarios as S

    g = golden("builds128")
    robot = L.RobotModel.from_dict(S.ARM6G)
    for i in robot.geometry_links:
        name = robot.links[i].name
        flat = np.asarray(L.build_link_sdf(robot.links[i].geometry, 0.64, 0.01, link_id=i).values).ravel(order="F")
        assert flat.size == 128 ** 3
        assert np.array_equal(flat[g[f"prim_{name}_idx"]], g[f"prim_{name}"]), name
        assert flat.astype(np.float64).sum() == float(g[f"prim_{name}_sum"]), name
    ico = L.TriangleMesh(g["mesh_V"], g["mesh_F"])
    flat = np.asarray(L.build_link_sdf(ico, 0.64, 0.01).values).ravel(order="F")
    got, want = flat[g["mesh_idx"]], g["mesh"]
    assert np.abs(got.astype(np.float64) - want).max() <= MESH_TOL
    assert np.mean(got == want) >= 0.999


def test_mlp_w128_tensor_cores_vs_cuda_cores(L):
    """Config 3 (iii) shape: W = 128 (V = 1,097,911, 3V = 3,293,733 outputs per
    rotation), hidden 32, 96 rotations: tcgen05 3xTF32 vs the CUDA-core kernel
    on every output, and vs numpy's sgemm (the reference's predict) on a slice."""
    import torch

    from oracle import linksdf_oracle as O

    grid = L.EnvGrid(1.28, 0.01)
    window = L.WindowGeometry.build(0.64, grid)
    V = window.n_masked
    assert V == 1_097_911
    rng = np.random.default_rng(128)
    model = L.TinyMlp.random(V, hidden=32, seed=128)
    R = L.sample_rotations(rng, 96)
    Rd = torch.from_numpy(R.reshape(-1, 9)).cuda()
    y_tc = model.predict_device(Rd, use_tensor_cores=True)
    y_cc = model.predict_device(Rd, use_tensor_cores=False)
    scale = float(torch.abs(y_cc).max().item())
    assert float(torch.abs(y_tc - y_cc).max().item()) <= 1e-5 * max(1.0, scale)
    cols = np.r_[0:6000, 3 * V - 6000:3 * V]
    want = O.mlp_predict(model.w1, model.b1, model.w2[:, cols], model.b2[cols], R[:8]).reshape(8, -1)
    got = y_tc[:8].cpu().numpy()[:, cols]
    assert np.abs(got - want).max() <= 1e-5 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("cloud", ["far_corners", "sparse_2k", "blobs", "empty"])
def test_config4_sparse_clouds_vs_dense(L, cloud):
    """The throughput batch (65,536 waypoints, segment bound and dilated-brick
    skip on) against clouds that leave most windows empty: == the dense gather
    on slices, and empty clouds give the clamp everywhere."""
    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG4
    robot, grid, sdfs, window = _setup(L, shape)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=5)
    rng = np.random.default_rng(5)
    if cloud == "far_corners":
        pts = S.far_crowd_cloud(200_000, 5)
    elif cloud == "sparse_2k":
        pts = S.sparse_cloud(2000, 5)
    elif cloud == "blobs":  # tight blobs: on brick boundaries, in a grid corner, near the base
        centres = np.array([[0.28, -0.28, 0.36], [-0.96, 0.96, -0.96], [0.12, 0.0, 0.44], [0.6, 0.6, -0.2]])
        pts = np.concatenate([c + rng.normal(0, 0.02, size=(300, 3)) for c in centres])
    else:
        pts = np.empty((0, 3))
    chk = L.DistanceChecker(robot, sdfs, grid, window).prepare(shape.n_waypoints, max(len(pts), 1), np.float32)
    d, link, voxel = _device_cycle(chk, q, np.asarray(pts, np.float32).reshape(-1, 3) if len(pts)
                                   else np.full((1, 3), np.nan, np.float32))
    if cloud == "empty":
        assert np.all(d == np.float32(chk.d_far_global)) and np.all(link == -1) and np.all(voxel == -1)
        return
    obs = L.voxelize_pointcloud(pts, grid)
    for a in (0, 40_000):
        part = L.TrajectorySdf.from_configs(robot, q[a:a + 2000], sdfs, grid, window)
        dense = L.RobotSdfBatch(part.device_values(), grid, part.d_far_global)
        dd, _, vd = L.query_min_distances(dense, obs, return_argmin=True)
        assert np.array_equal(dd, d[a:a + 2000]) and np.array_equal(vd, voxel[a:a + 2000])
        _, lp, _ = L.query_min_distances(part, obs, return_argmin=True)
        assert np.array_equal(lp, link[a:a + 2000])
    if cloud != "far_corners":
        assert np.any(link >= 0)  # some windows do see an obstacle


def test_sphere_baseline_vs_reference(L):
    """The covering-sphere comparator (query.py:254-291) on config 2's seed-21
    input against the reference's own output (tests/golden/sphere_c2.npz)."""
    import json

    from paper_2309_12543_b200 import scenarios as S

    g = golden("sphere_c2")
    shape = S.CONFIG2
    robot = L.RobotModel.from_dict(json.loads(bytes(g["robot_json"]).decode()))
    grid = L.EnvGrid(shape.grid_extent, shape.grid_res)
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=21)
    pts = S.cloud_for(shape, 21).astype(np.float32)
    assert np.array_equal(_digest(q), g["q_digest"]) and np.array_equal(_digest(pts), g["pts_digest"])
    poses = L.forward_kinematics_batch(robot, L.ConfigBatch(q))
    obs = L.voxelize_pointcloud(pts, grid)
    spheres = L.SphereRobotModel.from_robot(robot)
    d, st = L.sphere_baseline_distances(spheres, poses, obs, grid, return_stats=True)
    assert st["distance_evals"] == int(g["evals"])
    assert np.abs(d - g["d"]).max() <= 1e-12


def test_replay_end_to_end(L, tmp_path):
    """Config 5 replay (bench.py:410-430): manifest + f32 frame files -> one
    cycle per frame (direct and materialized) -> the distance CSV.  Both CSVs
    equal the one written from stream_min_distances on the same trajectory,
    and every frame matches the oracle on every 25th waypoint."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG5
    robot, grid, sdfs, window = _setup(L, shape)
    frames = S.moving_human_frames(12, shape.n_points, seed=5, dt=0.05)  # walks into range within the replay
    q = S.smooth_trajectory(shape.robot, shape.n_waypoints, seed=5)
    lines = []
    for k, (stamp, pts) in enumerate(frames):
        L.query.write_pointcloud_frame(tmp_path / f"f{k:03d}.bin", pts)
        lines.append(f"{stamp} f{k:03d}.bin")
    (tmp_path / "manifest.txt").write_text("# timestamp_ms frame\n" + "\n".join(lines) + "\n")
    out_d = L.run_replay(robot, sdfs, grid, window, q, tmp_path / "manifest.txt", tmp_path / "direct.csv")
    out_m = L.run_replay(robot, sdfs, grid, window, q, tmp_path / "manifest.txt", tmp_path / "mat.csv",
                         materialized=True)
    assert out_d["frames"] == 12 and out_d["waypoints"] == shape.n_waypoints and out_d["min_distance_m"] < 0.32
    traj = L.TrajectorySdf.from_configs(robot, q, sdfs, grid, window)
    rows = list(L.stream_min_distances(traj, L.query.iter_cloud_frames(tmp_path / "manifest.txt")))
    L.query.write_distance_csv(tmp_path / "stream.csv", rows, len(q))
    ref_csv = (tmp_path / "stream.csv").read_text()
    assert (tmp_path / "direct.csv").read_text() == ref_csv
    assert (tmp_path / "mat.csv").read_text() == ref_csv
    assert out_m["min_distance_m"] == out_d["min_distance_m"]
    grids = [s.values for s in sdfs]
    sub = np.arange(0, shape.n_waypoints, 25)
    near = 0
    for (stamp, d), (_, pts) in zip(rows, frames):
        rd, rl, _ = O.run_pipeline(shape.robot, q[sub], pts.astype(np.float32).astype(np.float64), shape.grid_extent,
                                   shape.grid_res, shape.link_extent, grids, [shape.link_res] * len(grids))
        assert np.abs(d[sub].astype(np.float64) - rd).max() <= D_TOL
        near += int((rl >= 0).any())
    assert near >= 3  # the human does come into range


def _linear_mlp(L, window, hidden=32):
    """A TinyMlp that IS the exact transform up to f32 rounding: units 0-8 / 9-17
    carry relu(+R) / relu(-R) (TinyMlp.initial), W2 maps them through the canonical
    points (y_vk = sum_j P_vj R_jk, approx.py:123-130 with placement.py:164)."""
    P = window.masked_points  # (V, 3)
    V = len(P)
    m = L.TinyMlp.initial(V, hidden=hidden, seed=0)
    w2 = np.zeros((hidden, 3 * V), np.float32)
    for j in range(3):
        for k in range(3):
            w2[3 * j + k, k::3] = P[:, j]
            w2[9 + 3 * j + k, k::3] = -P[:, j]
    return L.TinyMlp(m.w1, m.b1, w2, m.b2)


def test_neural_provider_honoured(L):
    """TrajectorySdf.from_poses with a NeuralTransformProvider places the windows
    with the MLP (no silent exact fallback): == the reference pipeline on the same
    windows (place_links_batch -> assemble -> gather), Appendix-B link on those
    windows, close to the oracle's neural pipeline and to the exact path; the
    MaterializedChecker honours the provider; DistanceChecker refuses it."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200 import scenarios as S

    shape = S.CONFIG2
    robot, grid, sdfs, window = _setup(L, shape)
    model = _linear_mlp(L, window)
    prov = L.NeuralTransformProvider(model, window)
    q = S.random_configs(shape.robot, 160, seed=8)
    pts = S.cloud_for(shape, 8)[:50_000]
    poses_all = L.forward_kinematics_batch(robot, L.ConfigBatch(q))
    gl = robot.geometry_links
    poses = L.LinkPoseBatch(rotations=poses_all.rotations[:, gl], translations=poses_all.translations[:, gl])
    obs = L.voxelize_pointcloud(pts, grid)
    traj = L.TrajectorySdf.from_poses(sdfs, poses, grid, prov)
    assert isinstance(traj, L.PlacedTrajectorySdf)
    d, link, voxel = L.query_min_distances(traj, obs, return_argmin=True)
    fields = list(L.place_links_batch(sdfs, poses, grid, prov))
    batch = L.assemble_robot_sdfs(((c, f) for c, _, f in fields), grid, len(q), traj.d_far_global)
    d2, _, v2 = L.query_min_distances(batch, obs, return_argmin=True)
    assert np.array_equal(d, d2) and np.array_equal(voxel, v2)
    win = {(c, li): f for c, li, f in fields}
    for c in range(len(q)):
        if link[c] < 0:
            continue
        v = obs.indices[voxel[c]]
        vals = []
        for li in range(len(gl)):
            rel = v - win[(c, li)].anchor
            inside = np.all(rel >= 0) and np.all(rel < window.dims)
            vals.append(win[(c, li)].values[tuple(rel)] if inside else np.inf)
        assert vals[link[c]] == d[c] and all(x != d[c] for x in vals[:link[c]])
    # the exact path (the model is the exact product up to f32 rounding)
    exact = L.TrajectorySdf.from_poses(sdfs, poses, grid, L.ExactTransformProvider(window))
    de = L.query_min_distances(exact, obs)
    assert np.abs(d.astype(np.float64) - de).max() <= 1e-5
    # the oracle's neural pipeline on a few configurations
    sub = np.arange(0, len(q), 20)
    e_r, r_r = shape.link_extent, shape.link_res
    env = O.Env(shape.grid_extent, shape.grid_res)
    anchors, dts, _ = O.align(poses.translations[sub].reshape(-1, 3), env, e_r)
    mask = O.window_mask(e_r, env).ravel(order="F")
    W = int(window.dims[0])
    wins = np.empty((len(sub), len(gl), W ** 3), np.float32)
    for i, c in enumerate(sub):
        for li in range(len(gl)):
            G = O.mlp_transform(model.w1, model.b1, model.w2, model.b2, poses.rotations[c, li],
                                dts[i * len(gl) + li], e_r)
            blk = np.full(W ** 3, np.float32(sdfs[li].d_far), np.float32)
            blk[mask] = O.trilinear(sdfs[li].values, e_r, r_r, (G * e_r).reshape(-1, 3))
            wins[i, li] = blk
    wins = wins.reshape(len(sub), len(gl), W, W, W).transpose(0, 1, 4, 3, 2)
    ob = O.assemble(wins, anchors.reshape(len(sub), len(gl), 3), env, traj.d_far_global)
    rd = O.query_min(ob, obs.indices, traj.d_far_global)
    assert np.abs(d[sub].astype(np.float64) - rd).max() <= 1e-5
    # MaterializedChecker with the provider; DistanceChecker refuses it
    mat = L.MaterializedChecker(robot, sdfs, grid, prov, q).prepare(len(pts), np.float32)
    dm, lm, vm = mat.query(pts.astype(np.float32))
    dn, ln, vn = L.query_min_distances(L.TrajectorySdf.from_poses(sdfs, poses, grid, prov),
                                       L.voxelize_pointcloud(pts.astype(np.float32), grid), return_argmin=True)
    assert np.array_equal(dm, dn) and np.array_equal(lm, ln) and np.array_equal(vm, vn)
    with pytest.raises(L.ValidationError):
        L.DistanceChecker(robot, sdfs, grid, prov)
    # query_trajectory with the provider: the same placed-window path
    d3, l3, v3 = L.query_trajectory(robot, q, sdfs, grid, prov, pts)
    assert np.array_equal(d3, d) and np.array_equal(l3, link) and np.array_equal(v3, voxel)


@pytest.mark.parametrize("n_cfg", [1, 37, 300])
def test_fused_neural_placement_matches_two_kernels(L, n_cfg):
    """lsdf_mlp_place (TinyMlp layer 2 on tcgen05 + trilinear epilogue, no G
    in HBM) == lsdf_mlp_predict(use_tensor_cores) -> lsdf_place_windows_g on
    the config-2 window (4.8k kept cells = 38 cell blocks), bit for bit: the
    same 3xTF32 MMA chain per output, the same f32 bias add and fp64 sampler.
    Rotation counts cover a partial tile, a tile spanning links and several tiles."""
    from paper_2309_12543_b200 import placement as P
    from paper_2309_12543_b200 import scenarios as S
    import paper_2309_12543_b200._native as N

    shape = S.CONFIG2
    robot, grid, sdfs, window = _setup(L, shape)
    rng = np.random.default_rng(n_cfg)
    H = 32
    model = L.TinyMlp(rng.normal(0, 0.5, (9, H)).astype(np.float32), rng.normal(0, 0.1, H).astype(np.float32),
                      rng.normal(0, 0.05, (H, 3 * window.n_masked)).astype(np.float32),
                      rng.normal(0, 0.2, 3 * window.n_masked).astype(np.float32))
    q = S.random_configs(shape.robot, n_cfg, seed=n_cfg)
    poses_all = L.forward_kinematics_batch(robot, L.ConfigBatch(q))
    gl = robot.geometry_links
    R = poses_all.rotations[:, gl]
    T = poses_all.translations[:, gl]
    from oracle import linksdf_oracle as O
    env = O.Env(shape.grid_extent, shape.grid_res)
    _, dt, _ = O.align(T.reshape(-1, 3), env, window.extent)
    t = N.torch()
    R_dev = N.to_device(np.ascontiguousarray(R.reshape(n_cfg, len(gl), 9)), t.float64)
    dt_dev = N.to_device(np.ascontiguousarray(dt.reshape(n_cfg, len(gl), 3)), t.float64)
    fused = P.place_windows_device(sdfs, R_dev, dt_dev, window, L.NeuralTransformProvider(model, window, fused=True))
    two = P.place_windows_device(sdfs, R_dev, dt_dev, window,
                                 L.NeuralTransformProvider(model, window, fused=False))
    a, b = fused.cpu().numpy(), two.cpu().numpy()
    assert a.shape == (n_cfg, len(gl), window.n_cells)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), np.abs(a - b).max()
