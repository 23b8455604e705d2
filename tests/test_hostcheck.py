"""CPU check of the kernels' scalar arithmetic against the reference goldens.

``tests/native/hostcheck.cpp`` compiles the SAME ``lsdf_math.cuh`` the CUDA
kernels use as host C++ (std::fma, -ffp-contract=off).  These tests pin the
operation orders (FMA chains where OpenBLAS uses them, plain mul/add where
numpy's elementwise loops do) without a GPU.  Test-only: the product never
loads this library.
"""

import ctypes
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from tests.conftest import REPO, golden

SRC = REPO / "tests" / "native" / "hostcheck.cpp"
LIB = REPO / "tests" / "native" / "_hostcheck.so"


@pytest.fixture(scope="module")
def hc():
    if not LIB.exists() or LIB.stat().st_mtime < max(SRC.stat().st_mtime,
                                                      (REPO / "paper_2309_12543_b200/csrc/lsdf_math.cuh").stat().st_mtime):
        subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", str(SRC),
                        "-o", str(LIB)], check=True)
    return ctypes.CDLL(str(LIB))


def P(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _robot(g):
    from paper_2309_12543_b200.robot import RobotModel

    return RobotModel.from_dict(json.loads(bytes(g["robot_json"]).decode()))


@pytest.mark.parametrize("name", ["scene_c1", "scene_small", "scene_arm7", "scene_c2"])
def test_fk_recipe(hc, name):
    g = golden(name)
    robot = _robot(g)
    table = robot.chain_table()
    q = np.ascontiguousarray(g["q"])
    C, L = len(q), robot.n_links
    R = np.zeros((C, L, 3, 3))
    T = np.zeros((C, L, 3))
    hc.hc_fk(table, L, P(q), ctypes.c_int64(C), robot.dof, P(R), P(T))
    assert np.abs(R - g["R"]).max() <= 1e-12 and np.abs(T - g["T"]).max() <= 1e-12
    # same glibc sin/cos as numpy in this image: bit-exact end to end
    assert np.array_equal(R, g["R"]) and np.array_equal(T, g["T"])


def _env(g):
    from paper_2309_12543_b200._native import EnvGridT

    e = EnvGridT()
    e.extent[:] = [float(g["env_extent"])] * 3
    e.resolution[:] = [float(g["env_res"])] * 3
    e.dims[:] = [int(round(2 * float(g["env_extent"]) / float(g["env_res"])))] * 3
    return e


@pytest.mark.parametrize("name", ["scene_c1", "scene_small", "scene_arm7", "scene_c2"])
def test_alignment_recipe(hc, name):
    g = golden(name)
    gl = g["geometry_links"]
    T = np.ascontiguousarray(g["T"][:, gl].reshape(-1, 3))
    W = (ctypes.c_int32 * 3)(*([int(round(2 * float(g["e_r"]) / float(g["env_res"])))] * 3))
    anchor = np.zeros((len(T), 3), np.int32)
    dt = np.zeros((len(T), 3))
    env = _env(g)
    bad = hc.hc_align(P(T), ctypes.c_int64(len(T)), ctypes.byref(env), W, P(anchor), P(dt))
    assert bad == 0
    assert np.array_equal(anchor.reshape(g["anchors"].shape), g["anchors"])
    # the reciprocal-multiply quotient (the FK kernels) gives the same bits
    anchor2, dt2 = np.zeros_like(anchor), np.zeros_like(dt)
    assert hc.hc_align_rinv(P(T), ctypes.c_int64(len(T)), ctypes.byref(env), W, P(anchor2), P(dt2)) == 0
    assert np.array_equal(anchor2, anchor) and np.array_equal(dt2, dt)


def test_shift_inverse_reciprocal_recipe(hc):
    rng = np.random.default_rng(3)
    n = 200_000
    R = np.ascontiguousarray(rng.normal(size=(n, 9)))
    dt = np.ascontiguousarray(rng.uniform(-0.05, 0.05, size=(n, 3)))
    hc.hc_shift_diff.restype = ctypes.c_double
    for e_r in (0.32, 0.3, 0.64, 0.17, 1.0 / 3.0):
        assert hc.hc_shift_diff(P(R), P(dt), ctypes.c_int64(n), ctypes.c_double(e_r)) == 0.0


def test_window_recipe_bit_exact(hc):
    """place_windows_kernel arithmetic == reference placement windows (stage isolation)."""
    from oracle import linksdf_oracle as O

    g = golden("scene_small")
    gl = g["geometry_links"]
    e_r, r_r = float(g["e_r"]), float(g["r_r"])
    env = O.Env(float(g["env_extent"]), float(g["env_res"]))
    W = O.window_width(e_r, env)
    Pt = np.zeros((3, int(W.max())))
    for a in range(3):
        Pt[a, : W[a]] = (np.arange(W[a]) - W[a] // 2) * env.resolution[a] / e_r
    mask = np.ascontiguousarray(O.window_mask(e_r, env).ravel(order="F").astype(np.uint8))
    Rg = g["R"][:, gl]
    anchors, deltas, _ = O.align(g["T"][:, gl].reshape(-1, 3), env, e_r)
    deltas = deltas.reshape(Rg.shape[0], Rg.shape[1], 3)
    out = np.zeros(int(np.prod(W)), np.float32)
    Wc = (ctypes.c_int32 * 3)(*W.tolist())
    mismatches = 0
    for c in range(Rg.shape[0]):
        for li in range(Rg.shape[1]):
            grid = np.ascontiguousarray(np.ravel(g["grids"][li], order="F"))
            dims = (ctypes.c_int32 * 3)(*g["grids"][li].shape)
            ext = (ctypes.c_double * 3)(e_r, e_r, e_r)
            res = (ctypes.c_double * 3)(r_r, r_r, r_r)
            R = np.ascontiguousarray(Rg[c, li])
            dt = np.ascontiguousarray(deltas[c, li])
            hc.hc_window(P(R), P(dt), P(grid), dims, ext, res, ctypes.c_float(e_r), P(Pt), int(W.max()), Wc,
                         P(mask), ctypes.c_double(e_r), P(out))
            ref = np.ravel(g["windows"][c, li], order="F")
            mismatches += int(np.sum(out != ref))
    assert mismatches == 0


def test_trilinear_recipe(hc):
    t = golden("trilinear")
    grid = np.ascontiguousarray(np.ravel(t["values"], order="F"))
    dims = (ctypes.c_int32 * 3)(*t["values"].shape)
    e, r = float(t["extent"]), float(t["res"])
    pts = np.ascontiguousarray(t["pts"])
    out = np.zeros(len(pts), np.float32)
    hc.hc_trilinear(P(grid), dims, (ctypes.c_double * 3)(e, e, e), (ctypes.c_double * 3)(r, r, r),
                    ctypes.c_float(e), P(pts), ctypes.c_int64(len(pts)), P(out))
    assert np.array_equal(out, t["out"])


def _prim_params(geom):
    p = np.zeros(8)
    if geom["type"] == "sphere":
        p[0] = geom["radius"]
        p[1:4] = geom.get("center", (0, 0, 0))
        return 0, p
    if geom["type"] == "capsule":
        ax = np.asarray(geom.get("axis", (0, 0, 1.0)), dtype=np.float64)
        p[0], p[1] = geom["radius"], geom["half_length"]
        p[2:5] = ax / np.linalg.norm(ax)
        return 1, p
    p[0:3] = geom["half_extents"]
    return 2, p


def test_primitive_recipe(hc):
    b = golden("builds")
    for key in [k for k in b.files if k.startswith("prim_") and not k.endswith("_json")]:
        geom = json.loads(bytes(b[key + "_json"]).decode())
        kind, prm = _prim_params(geom)
        dims = b[key].shape
        out = np.zeros(int(np.prod(dims)), np.float32)
        hc.hc_primitive_grid(kind, P(prm), (ctypes.c_double * 3)(0.2, 0.2, 0.2),
                             (ctypes.c_double * 3)(0.01, 0.01, 0.01), (ctypes.c_int32 * 3)(*dims), P(out))
        assert np.array_equal(out, np.ravel(b[key], order="F")), key


def test_mesh_recipe(hc):
    b = golden("builds")
    for name in ("ico", "box", "tiltbox", "open"):
        V, F = b[f"mesh_{name}_V"], b[f"mesh_{name}_F"]
        e, r = b[f"mesh_{name}_er"]
        tri = np.ascontiguousarray(np.concatenate([V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]], axis=1))
        dims = b[f"mesh_{name}"].shape
        out = np.zeros(int(np.prod(dims)), np.float32)
        hc.hc_mesh_grid(P(tri), len(tri), int(name != "open"), (ctypes.c_double * 3)(e, e, e),
                        (ctypes.c_double * 3)(r, r, r), (ctypes.c_int32 * 3)(*dims), P(out))
        ref = np.ravel(b[f"mesh_{name}"], order="F")
        assert np.abs(out - ref).max() <= 1e-5, name   # SURVEY §8c mesh tolerance
        assert np.array_equal(out, ref), name


def test_mlp_recipe(hc):
    m = golden("mlp")
    R = np.ascontiguousarray(m["R"].reshape(-1, 9))
    n_out = m["w2"].shape[1]
    y = np.zeros((len(R), n_out), np.float32)
    hc.hc_mlp(P(np.ascontiguousarray(m["w1"])), P(np.ascontiguousarray(m["b1"])), P(np.ascontiguousarray(m["w2"])),
              P(np.ascontiguousarray(m["b2"])), m["w1"].shape[1], ctypes.c_int64(n_out), P(R),
              ctypes.c_int64(len(R)), P(y))
    ref = m["predict"].reshape(len(R), -1)
    assert np.abs(y - ref).max() <= 1e-5
    print("mlp bit-exact fraction", np.mean(y == ref))
