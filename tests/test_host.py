"""CPU-only tests: the C-ABI library loads and exports the header, host-side
tables are right, and the product fails loudly without a GPU (no CPU path)."""

import ctypes
import re

import numpy as np
import pytest

from tests.conftest import REPO


def test_library_exports_every_header_symbol():
    from paper_2309_12543_b200 import _native as N
    from paper_2309_12543_b200.build import build

    build()
    lib = ctypes.CDLL(str(N.LIB_PATH))
    header = (REPO / "include" / "linksdf_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t|uint64_t|const char\*)\s+(lsdf_\w+)\s*\(", header, re.M))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(N.EXPORTS) == declared
    N.load_library()
    assert b"sm_100a" in N.lib().lsdf_version()


def test_ctypes_struct_layouts_match_header():
    from paper_2309_12543_b200 import _native as N

    # sizes implied by include/linksdf_b200.h on LP64
    assert ctypes.sizeof(N.EnvGridT) == 64
    assert ctypes.sizeof(N.LinkT) == 16 + 45 * 8
    assert ctypes.sizeof(N.LinkGridT) == 8 + 8 + 12 + 4 + 48 + 4 + 36
    assert ctypes.sizeof(N.WindowT) == 16 + 8 + 8 + 8 + 8 + 8 + 8 + 8


def test_sass_is_sm100a():
    import subprocess

    from paper_2309_12543_b200 import _native as N

    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2309_12543_b200 as L

    grid = L.EnvGrid(1.0, 0.1)
    with pytest.raises(L.LinkSdfError):
        L.voxelize_pointcloud(np.zeros((4, 3)), grid)
    with pytest.raises(L.LinkSdfError):
        L.build_link_sdf(L.Sphere(0.1), 0.2, 0.05)


def test_window_tables_match_mask():
    import paper_2309_12543_b200 as L

    for res, e in ((0.04, 0.32), (0.1, 0.3), (0.04, 1.2), (0.01, 0.64)):
        grid = L.EnvGrid(1.0 if res > 0.01 else 1.28, res)
        w = L.WindowGeometry.build(e, grid)
        W = w.dims
        m = w.mask
        for mx in range(0, W[0], max(1, W[0] // 7)):
            for my in range(W[1]):
                zs = np.nonzero(m[mx, my])[0]
                if len(zs):
                    assert zs[-1] + 1 - zs[0] == len(zs)  # ball rows are intervals along z
    w = L.WindowGeometry.build(0.32, L.EnvGrid(1.0, 0.04))
    assert w.n_masked == 2103  # SURVEY §8 probe


def test_chain_table_constants():
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    robot = L.RobotModel.from_dict(S.ARM7G)
    t = robot.chain_table()
    assert robot.dof == 7 and robot.n_links == 8 and robot.geometry_links == list(range(1, 8))
    assert t[0].kind == 0 and t[1].kind == 1 and t[7].geom_slot == 6 and t[7].parent == 6
    j2 = robot.joint("j2")
    assert np.array_equal(np.array(t[2].joint_R[:]).reshape(3, 3), j2.origin.rotation)


def test_validation_errors_host_side():
    import paper_2309_12543_b200 as L

    with pytest.raises(L.ValidationError):
        L.EnvGrid(1.0, 0.3)
    with pytest.raises(L.ValidationError):
        L.window_dims(0.25, L.EnvGrid(1.0, 0.1))
    with pytest.raises(L.ValidationError):
        L.canonical_points([0.3, 0.3, 0.2], L.EnvGrid(1.0, 0.1))
    with pytest.raises(L.ValidationError):
        L.masked_window_points(5)
    g = L.EnvGrid(1.0, 0.1)
    with pytest.raises(L.ValidationError):
        L.assemble_robot_sdfs([], g, 10_000_000, 0.5, max_bytes=1 << 20)


def test_c_abi_client_builds_and_fails_loudly(tmp_path):
    """The plain-C client (tests/native/abi_demo.c) links against the library alone, reads a scene
    written from the host recipes, and without a GPU exits non-zero with a CUDA error (no CPU path)."""
    import subprocess

    import torch

    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S
    from paper_2309_12543_b200.build import build_demo
    from tests.native.abi_scene import write_scene

    exe = build_demo()
    robot = L.RobotModel.from_dict(S.ARM7G)
    grid = L.EnvGrid(1.0, 0.04)
    ax = -0.32 + (np.arange(16) + 0.5) * 0.04
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    sdfs = [L.LinkSdf(0.32, 0.04, np.sqrt(X * X + Y * Y + Z * Z) - 0.05, link_id=i) for i in robot.geometry_links]
    window = L.WindowGeometry.build(0.32, grid)
    q = np.zeros((8, robot.dof))
    scene = tmp_path / "scene.bin"
    write_scene(scene, robot, sdfs, grid, window, q, np.zeros((5, 3), np.float32))
    raw = scene.read_bytes()
    assert raw[:8] == b"LSDFABI1"
    assert int.from_bytes(raw[8:16], "little") == 32  # header section
    if torch.cuda.is_available():
        pytest.skip("GPU present: tests/test_gpu_parity.py::test_c_abi_client covers the run")
    r = subprocess.run([str(exe), str(scene), str(tmp_path / "out.bin")], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0 and "cuda" in r.stderr.lower()


def test_scan_bounds_hold_on_random_grids():
    """The early-stop and segment bounds the shell scan relies on (LinkSdf.core_radius,
    LinkSdf.segment_bound: lower bounds by convexity, upper bound + |h|/2) hold for
    trilinear samples of noisy and exact grids, checked with the oracle's trilinear."""
    from oracle import linksdf_oracle as O
    from paper_2309_12543_b200.grids import LinkSdf, interpolation_spread

    rng = np.random.default_rng(5)
    # the spread itself: sum_i w_i |v_i - p| <= |h| / 2 over random cell fractions and anisotropic h
    h = np.array([0.01, 0.02, 0.015])
    f = rng.random((20000, 3))
    corners = np.array([[i, j, k] for k in (0, 1) for j in (0, 1) for i in (0, 1)], dtype=np.float64)
    w = np.prod(np.where(corners[None], f[:, None], 1.0 - f[:, None]), axis=-1)
    dist = np.linalg.norm((corners[None] - f[:, None]) * h, axis=-1)
    assert (w * dist).sum(axis=1).max() <= interpolation_spread(h) * (1 + 1e-12)
    for shape_kind, noise in (("capsule", 0.004), ("sphere", 0.004), ("capsule", 0.0)):
        e_r, r_r = 0.16, 0.01
        c = -e_r + (np.arange(32) + 0.5) * r_r
        X, Y, Z = np.meshgrid(c, c, c, indexing="ij")
        if shape_kind == "capsule":
            t = np.clip(Z, -0.05, 0.05)
            base = np.sqrt(X * X + Y * Y + (Z - t) ** 2) - 0.04
        else:
            base = np.sqrt(X * X + Y * Y + Z * Z) - 0.05
        # noise 0: an exact distance grid, where the interpolation term of the upper bound is tight
        vals = (base + rng.normal(0, noise, base.shape)).astype(np.float32)
        sdf = LinkSdf(e_r, r_r, vals, link_id=0)
        kappa = sdf.core_radius()
        a, u, length, k_lo, k_hi = sdf.segment_bound()
        pts = rng.uniform(c[0], c[-1], size=(40000, 3))
        v = O.trilinear(sdf.values, e_r, r_r, pts).astype(np.float64)
        assert np.all(v >= np.linalg.norm(pts, axis=1) - kappa)
        a, u_seg = np.asarray(a), np.asarray(u)
        tt = np.clip((pts - a) @ u_seg, 0.0, length)
        d = np.linalg.norm(pts - a - tt[:, None] * u_seg, axis=1)
        assert np.all(v >= d - k_lo) and np.all(v <= d + k_hi)
        # Window cells reach |p| <= e_r + |dt|, past the hull of the cell centres,
        # where the sample is the far value: the lower bounds still hold as
        # min(bound, d_far) (values >= the clamp never change a minimum), but
        # the upper bound holds only inside the hull -- the kernel applies it to
        # chunks whose shell radius + |dt| stays in the inscribed ball.
        hull = e_r - r_r / 2
        u = rng.normal(size=(60000, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        pts = u * (e_r + 0.04) * np.cbrt(rng.random((60000, 1)))
        v = O.trilinear(sdf.values, e_r, r_r, pts).astype(np.float64)
        rad = np.linalg.norm(pts, axis=1)
        tt = np.clip((pts - a) @ u_seg, 0.0, length)
        d = np.linalg.norm(pts - a - tt[:, None] * u_seg, axis=1)
        assert np.all(v >= np.minimum(rad - kappa, sdf.d_far))
        assert np.all(v >= np.minimum(d - k_lo, sdf.d_far))
        ball = rad <= hull - 1e-5
        assert np.all(v[ball] <= d[ball] + k_hi)
        outside = np.any(np.abs(pts) > hull, axis=1)
        assert np.any(v[outside] > d[outside] + k_hi)  # why the guard exists (not vacuous)


def test_segment_bound_quadratic_form():
    """The scan's f32 segment distance (lsdf_query.cu seg_d2: |q|^2 - s^2 + (s - t)^2
    from per-task constants 2 A b, |b|^2, A u, b.u and per-cell sigma^2 |m'|^2, with
    fma emulated as one rounding of the exact fp64 product-sum) stays within
    SEG_D2_ERR / 4 = 2^-23 m^2 of the exact squared distance, over random rotations,
    window residuals, segments and every window cell."""
    f32 = np.float32
    rng = np.random.default_rng(11)

    def fma(a, b, c):
        return f32(np.float64(a) * np.float64(b) + np.float64(c))

    n, W, e_r, r_e = 300_000, 16, 0.32, 0.04
    P = (np.arange(W) - W // 2) * r_e / e_r
    qn = rng.normal(size=(n, 4))
    qn /= np.linalg.norm(qn, axis=1, keepdims=True)
    w, x, y, z = qn.T
    R = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
                  2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                  2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], 1).reshape(n, 3, 3)
    dtinv = rng.uniform(-0.1, 0.1, (n, 3))
    a3 = rng.uniform(-0.12, 0.12, (n, 3)).astype(f32).astype(np.float64)
    u = rng.normal(size=(n, 3))
    u = (u / np.linalg.norm(u, axis=1, keepdims=True)).astype(f32).astype(np.float64)
    L = rng.uniform(0, 0.25, n).astype(f32)
    m = rng.integers(0, W, (n, 3))
    c = W // 2
    # exact: the fp64 link-frame point (placement.py:164-167) minus the segment origin
    q = e_r * (np.einsum("na,nak->nk", P[m], R) + dtinv) - a3
    s_ex = np.einsum("nk,nk->n", q, u)
    t_ex = np.clip(s_ex, 0, L.astype(np.float64))
    d2_ex = np.sum((q - t_ex[:, None] * u) ** 2, axis=1)
    # the kernel's constants (shell_setup) and evaluation (seg_cell, seg_d2)
    f = e_r * (P[1] - P[0])
    b = e_r * dtinv - a3 + e_r * np.einsum("a,nak->nk", np.full(3, P[c]), R)
    sw = np.concatenate([2 * f * np.einsum("nak,nk->na", R, b), np.sum(b * b, 1)[:, None]], 1).astype(f32)
    sv = np.concatenate([f * np.einsum("nak,nk->na", R, u), np.sum(b * u, 1)[:, None]], 1).astype(f32)
    s2 = f32(f * f)
    px, py, pz = [(m[:, i] - c).astype(f32) for i in range(3)]
    mm = fma(px, f32(px * s2), fma(py, f32(py * s2), f32(f32(pz * pz) * s2)))
    qq = fma(pz, sw[:, 2], fma(py, sw[:, 1], fma(px, sw[:, 0], f32(mm + sw[:, 3]))))
    sp = fma(pz, sv[:, 2], fma(py, sv[:, 1], fma(px, sv[:, 0], sv[:, 3])))
    dd = f32(sp - np.minimum(np.maximum(sp, f32(0)), L))
    d2 = np.maximum(fma(dd, dd, fma(-sp, sp, qq)), f32(0))
    assert np.abs(d2.astype(np.float64) - d2_ex).max() <= 2.0 ** -23


def test_link_major_threshold_matches_fk_crossover():
    """The checker keeps poses link-major from the batch size at which FK runs one
    thread per configuration (the kernel whose writes the layout serves)."""
    from paper_2309_12543_b200.checker import LINK_MAJOR_MIN

    src = (REPO / "paper_2309_12543_b200" / "csrc" / "lsdf_fk.cu").read_text()
    m = re.search(r"constexpr int64_t FK_SERIAL_MIN = (\d+);", src)
    assert m and int(m.group(1)) == LINK_MAJOR_MIN
    header = (REPO / "include" / "linksdf_b200.h").read_text()
    from paper_2309_12543_b200 import _native as N

    assert f"#define LSDF_QUERY_BY_POSITION {N.QUERY_BY_POSITION}" in header
    assert f"#define LSDF_QUERY_POSES_LINK_MAJOR {N.QUERY_POSES_LINK_MAJOR}" in header


def test_exact_only_checker_refuses_other_providers():
    """DistanceChecker runs the exact transform in its fused cycle: a neural (or any
    other) provider is refused before any GPU work, never silently replaced."""
    import paper_2309_12543_b200 as L
    from paper_2309_12543_b200 import scenarios as S

    robot = L.RobotModel.from_dict(S.ARM6G)
    grid = L.EnvGrid(1.0, 0.04)
    window = L.WindowGeometry.build(0.32, grid)
    model = L.TinyMlp.initial(window.n_masked, hidden=32)
    prov = L.NeuralTransformProvider(model, window)
    ax = -0.32 + (np.arange(16) + 0.5) * 0.04
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    sdfs = [L.LinkSdf(0.32, 0.04, np.sqrt(X * X + Y * Y + Z * Z) - 0.05, link_id=i) for i in robot.geometry_links]
    with pytest.raises(L.ValidationError, match="exact transform"):
        L.DistanceChecker(robot, sdfs, grid, prov)
    L.checker._require_exact(window, "x")
    L.checker._require_exact(L.ExactTransformProvider(window), "x")


def test_replay_frame_reader(tmp_path):
    """run_replay's reader: a frame's f32 points straight into a (cap, 3) buffer, NaN past them."""
    from paper_2309_12543_b200 import query as Q
    from paper_2309_12543_b200 import replay as R
    from paper_2309_12543_b200.errors import ValidationError

    pts = np.float64([[0.1, -0.2, 0.3], [1.5, 2.5, -3.5], [0.0, 0.0, 1e-3]])
    f = tmp_path / "f.bin"
    Q.write_pointcloud_frame(f, pts)
    buf = np.zeros((5, 3), np.float32)
    assert R.frame_point_count(f) == 3 and R.read_frame_into(f, buf) == 3
    assert np.array_equal(buf[:3], pts.astype(np.float32)) and np.all(np.isnan(buf[3:]))
    with pytest.raises(ValidationError):
        R.read_frame_into(f, np.zeros((2, 3), np.float32))
    f.write_bytes(f.read_bytes()[:-4])
    with pytest.raises(ValidationError):
        R.read_frame_into(f, buf)
