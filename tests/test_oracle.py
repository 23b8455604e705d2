"""Pin the CPU oracle against the reference's golden fixtures (CPU only).

The oracle (``oracle/linksdf_oracle.py``) is the checker the GPU parity tests
and the bench's CPU baseline use on the GPU box; here it must reproduce the
reference outputs stored by ``tests/golden/make_golden.py``.  Reference
known-answer tests it restates are cited per test.
"""

import json

import numpy as np
import pytest

from oracle import linksdf_oracle as O
from tests.conftest import golden


def _doc(g):
    return json.loads(bytes(g["robot_json"]).decode())


@pytest.mark.parametrize("name", ["scene_c1", "scene_small", "scene_arm7", "scene_c2"])
def test_fk_matches_reference(name):
    g = golden(name)
    R, T = O.fk(O.chain_from_doc(_doc(g)), g["q"])
    # robot.py:305-347; reference's own bar is 1e-12 (test_robot.py:168)
    assert np.abs(R - g["R"]).max() <= 1e-12
    assert np.abs(T - g["T"]).max() <= 1e-12
    assert np.array_equal(R, g["R"]) and np.array_equal(T, g["T"])


@pytest.mark.parametrize("name", ["scene_c1", "scene_small"])
def test_full_pipeline_bit_exact(name):
    g = golden(name)
    grids = list(g["grids"])
    out = O.run_pipeline(_doc(g), g["q"], g["points"], float(g["env_extent"]),
                         float(g["env_res"]), float(g["e_r"]), grids,
                         [float(g["r_r"])] * len(grids), return_all=True)
    assert np.array_equal(out["anchors"], g["anchors"])
    assert np.array_equal(out["indices"], g["indices"])
    assert out["n_dropped"] == int(g["n_dropped"])
    assert np.array_equal(out["d"], g["d"])
    assert np.array_equal(out["link"], g["link"])
    assert np.array_equal(out["voxel"], g["voxel"])
    if "windows" in g:
        assert np.array_equal(out["windows"], g["windows"])
    if "batch" in g:
        assert np.array_equal(out["batch"], g["batch"])
    env = O.Env(float(g["env_extent"]), float(g["env_res"]))
    pl = O.per_link_min(out["windows"], out["anchors"], out["indices"],
                        [float(g["e_r"])] * len(grids), float(g["d_far_global"]))
    assert np.array_equal(pl, g["per_link"])
    assert env.dims.prod() > 0


def test_grids_match_reference_builds():
    g = golden("scene_c1")
    doc = _doc(g)
    chain = O.chain_from_doc(doc)
    gl = O.geometry_links(chain)
    for k, li in enumerate(gl):
        grid = O.build_grid(chain[li]["geometry"], float(g["e_r"]), float(g["r_r"]))
        assert np.array_equal(grid, g["grids"][k])


def test_primitive_and_mesh_builds():
    b = golden("builds")
    for key in [k for k in b.files if k.startswith("prim_") and not k.endswith("_json")]:
        geom = json.loads(bytes(b[key + "_json"]).decode())
        assert np.array_equal(O.build_grid(geom, 0.2, 0.01), b[key]), key
    for name in ("ico", "box", "tiltbox", "open"):
        V, F = b[f"mesh_{name}_V"], b[f"mesh_{name}_F"]
        e, r = b[f"mesh_{name}_er"]
        signed = name != "open"
        got = O.build_grid(None, e, r, mesh=(V, F, signed))
        # meshes: SURVEY §8c allows 1e-5 m; the restatement is bit-exact here
        assert np.abs(got - b[f"mesh_{name}"]).max() <= 1e-5, name
        assert np.array_equal(got, b[f"mesh_{name}"]), name


def test_known_answer_tie_and_clamp():
    k = golden("known_answer")
    env = O.Env(1.0, 0.1)
    grids = list(k["grids"])
    windows, anchors = O.place_windows(grids, [0.3, 0.3], [0.01, 0.01], k["R"], k["T"], env, 0.3)
    batch = O.assemble(windows, anchors, env, 0.3)
    for name in ("tie", "far", "empty"):
        d, link, voxel = O.argmin_oracle(batch, windows, anchors, k[f"{name}_indices"], 0.3)
        assert np.array_equal(d, k[f"{name}_d"])
        assert np.array_equal(link, k[f"{name}_link"])
        assert np.array_equal(voxel, k[f"{name}_voxel"])
    # SURVEY Appendix B literal values
    assert np.allclose(k["tie_d"], [0.08012503, 0.08012503])
    assert list(k["tie_link"]) == [0, 0] and list(k["tie_voxel"]) == [0, 0]
    assert list(k["far_link"]) == [-1, -1] and np.all(k["far_d"] == np.float32(0.3))


def test_trilinear_matches_reference():
    t = golden("trilinear")
    out = O.trilinear(t["values"], float(t["extent"]), float(t["res"]), t["pts"])
    assert np.array_equal(out, t["out"])


def test_mlp_matches_reference():
    m = golden("mlp")
    y = O.mlp_predict(m["w1"], m["b1"], m["w2"], m["b2"], m["R"])
    assert np.array_equal(y, m["predict"])
    g = O.mlp_transform(m["w1"], m["b1"], m["w2"], m["b2"], m["R"], m["dt"], 0.3)
    assert np.array_equal(g, m["infer"])
    ex = O.transform_exact(m["R"], m["dt"], 0.3, m["masked_points"])
    assert np.array_equal(ex, m["exact"])


# -- reference known-answer tests restated on the oracle ---------------------

def test_alignment_known_answers():
    # test_placement.py:55-87
    env = O.Env(1.0, 0.1)
    a, d, _ = O.align(np.float64([[0.05, 0.05, 0.05]]), env, 0.3)
    assert list(a[0]) == [7, 7, 7] and np.allclose(d, 0, atol=1e-15)
    a, d, _ = O.align(np.float64([[0.07, 0.05, 0.05]]), env, 0.3)
    assert list(a[0]) == [7, 7, 7] and np.allclose(d, [[0.02, 0, 0]], atol=1e-15)
    a, d, _ = O.align(np.float64([[0.10, 0.05, 0.05]]), env, 0.3)
    assert list(a[0]) == [8, 7, 7] and np.allclose(d, [[-0.05, 0, 0]], atol=1e-15)
    a, _, bad = O.align(np.float64([[1.05, 0.0, 0.0], [1.7, 0.0, 0.0]]), env, 0.3)
    assert list(a[0]) == [17, 7, 7] and list(bad) == [False, True]


def test_voxelize_known_answers():
    # test_query.py:105-136, test_grids.py:43-69
    env = O.Env(1.0, 0.1)
    idx, n, drop = O.voxelize(np.tile(np.float64([0.31, 0.02, -0.44]), (1000, 1)), env)
    assert len(idx) == 1 and n == 1000 and drop == 0
    idx, n, drop = O.voxelize(np.float64([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0], [0.0, -3.0, 0.0]]), env)
    assert len(idx) == 1 and drop == 2 and list(idx[0]) == [10, 10, 10]
    idx, _, drop = O.voxelize(np.float64([[1.0, 0, 0], [-1.0, 0, 0]]), env)
    assert drop == 1 and list(idx[0]) == [0, 10, 10]


# ----------------------------------------------------------------------------- round-2 fixtures: the benchmarked inputs


def _bench_grids(shape):
    chain = O.chain_from_doc(shape.robot)
    return [O.build_grid(chain[i]["geometry"], shape.link_extent, shape.link_res) for i in O.geometry_links(chain)]


def test_oracle_on_bench_config2_seed21():
    """The oracle reproduces the reference on bench.py's own config-2 input (seed 21, 500 waypoints)."""
    from paper_2309_12543_b200 import scenarios as S

    g = golden("bench_c2")
    shape = S.CONFIG2
    q = S.random_configs(shape.robot, shape.n_waypoints, seed=21)
    pts = S.cloud_for(shape, 21).astype(np.float32)
    assert np.array_equal(np.float64([q.sum(), np.abs(q).sum(), q.size]), g["s21_q_digest"])
    d, link, voxel = O.run_pipeline(shape.robot, q, pts, shape.grid_extent, shape.grid_res, shape.link_extent,
                                    _bench_grids(shape), [shape.link_res] * 6)
    assert np.array_equal(d, g["s21_d"]) and np.array_equal(link, g["s21_link"])
    assert np.array_equal(voxel, g["s21_voxel"])


def test_oracle_builds_at_128():
    """Config 3 (i): an arm6g capsule at 128^3 and the 1,280-triangle icosphere (strided cells)."""
    from paper_2309_12543_b200 import scenarios as S

    g = golden("builds128")
    geo = next(lk for lk in S.ARM6G["links"] if lk["name"] == "l2")["geometry"]
    flat = O.build_grid(geo, 0.64, 0.01).ravel(order="F")
    assert np.array_equal(flat[g["prim_l2_idx"]], g["prim_l2"])
    ijk = np.stack(np.unravel_index(g["mesh_idx"][::10], (128, 128, 128), order="F"), axis=1)
    got = O.mesh_sdf(g["mesh_V"], g["mesh_F"], -0.64 + (ijk + 0.5) * 0.01, signed=True).astype(np.float32)
    assert np.array_equal(got, g["mesh"][::10])
