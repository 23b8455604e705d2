"""Seeded synthetic inputs for the five measured configurations.

Nothing here is on the hot path: these builders only produce robot JSON
documents, joint-space trajectories and obstacle point clouds of the shapes
BASELINE.json names, so the bench, the tests and the golden-vector script all
draw the same inputs from ``np.random.default_rng(seed)``.

* ``ARM6G`` — the reference test suite's 6-DoF chain (``tests/conftest.py:73-117``)
  with primitive collision geometry on l1..l6 (capsules, a box, a sphere).
* ``ARM7G`` — ARM6G plus a 7th revolute joint about x carrying a small sphere.
* ``human_cloud`` — 90 % anisotropic Gaussian blob + 10 % uniform clutter over
  [-1, 1)^3, deliberately NOT clipped: out-of-grid points are dropped and
  counted by ``voxelize_pointcloud`` as the reference does (``query.py:112,124``).
* ``crowd_cloud`` — ten blobs without clutter (config 4).
* ``moving_human_frames`` — one 30k-point blob walking toward the base at
  1.6 m/s, sampled every 8 ms (config 5, ``PAPER.md:304``).
"""

from __future__ import annotations

import copy
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_ARM6_KINEMATICS = {
    "name": "arm6g",
    "link_reach": 0.6,
    "links": [
        {"name": "base"},
        {"name": "l1", "parent_joint": "j1"},
        {"name": "l2", "parent_joint": "j2", "origin": {"xyz": [0, 0, 0.125]}},
        {"name": "l3", "parent_joint": "j3", "origin": {"xyz": [0.01, 0, 0.21]}},
        {"name": "l4", "parent_joint": "j4", "origin": {"xyz": [-0.01, 0, 0.0]}},
        {"name": "l5", "parent_joint": "j5", "origin": {"xyz": [0, 0, 0.07]}},
        {"name": "l6", "parent_joint": "j6", "origin": {"xyz": [0, 0, 0.04]}},
    ],
    "joints": [
        {"name": "j1", "type": "revolute", "parent_link": "base",
         "origin": {"xyz": [0, 0, 0.148]}, "axis": [0, 0, 1],
         "limits": {"position": [-2.967, 2.967], "velocity": 3.92, "acceleration": 19.6}},
        {"name": "j2", "type": "revolute", "parent_link": "l1",
         "origin": {"xyz": [0.03, 0, 0.047], "rpy": [0, 0, 0.1]}, "axis": [0, 1, 0],
         "limits": {"position": [-2.094, 2.094], "velocity": 2.62, "acceleration": 13.1}},
        {"name": "j3", "type": "revolute", "parent_link": "l2",
         "origin": {"xyz": [0, 0, 0.085], "rpy": [0.05, 0, 0]}, "axis": [0, 1, 0],
         "limits": {"position": [-2.181, 2.792], "velocity": 2.79, "acceleration": 13.95}},
        {"name": "j4", "type": "revolute", "parent_link": "l3",
         "origin": {"xyz": [0, 0.02, 0.1]}, "axis": [0, 0, 1],
         "limits": {"position": [-3.316, 3.316], "velocity": 3.92, "acceleration": 19.6}},
        {"name": "j5", "type": "revolute", "parent_link": "l4",
         "origin": {"xyz": [0, 0, 0.08], "rpy": [0, -0.2, 0]}, "axis": [0, 1, 0],
         "limits": {"position": [-2.094, 2.094], "velocity": 3.02, "acceleration": 15.1}},
        {"name": "j6", "type": "revolute", "parent_link": "l5",
         "origin": {"xyz": [0, 0, 0.044]}, "axis": [0, 0, 1],
         "limits": {"position": [-6.283, 6.283], "velocity": 4.71, "acceleration": 23.55}},
    ],
}

_ARM6_GEOMETRY = {
    "l1": {"type": "capsule", "radius": 0.07, "half_length": 0.06},
    "l2": {"type": "capsule", "radius": 0.06, "half_length": 0.08},
    "l3": {"type": "capsule", "radius": 0.05, "half_length": 0.07},
    "l4": {"type": "capsule", "radius": 0.045, "half_length": 0.05},
    "l5": {"type": "box", "half_extents": [0.04, 0.04, 0.05]},
    "l6": {"type": "sphere", "radius": 0.05},
}


def _with_geometry(doc: dict, geometry: dict) -> dict:
    out = copy.deepcopy(doc)
    for link in out["links"]:
        if link["name"] in geometry:
            link["geometry"] = copy.deepcopy(geometry[link["name"]])
    return out


ARM6G = _with_geometry(_ARM6_KINEMATICS, _ARM6_GEOMETRY)

ARM7G = copy.deepcopy(ARM6G)
ARM7G["name"] = "arm7g"
ARM7G["links"].append(
    {"name": "l7", "parent_joint": "j7", "origin": {"xyz": [0, 0, 0.03]},
     "geometry": {"type": "sphere", "radius": 0.04}}
)
ARM7G["joints"].append(
    {"name": "j7", "type": "revolute", "parent_link": "l6",
     "origin": {"xyz": [0, 0, 0.05]}, "axis": [1, 0, 0],
     "limits": {"position": [-3.0, 3.0], "velocity": 4.71, "acceleration": 23.55}}
)

HUMAN_CENTER = (0.45, 0.0, 0.3)
HUMAN_SIGMA = (0.10, 0.15, 0.30)


def write_robot(doc: dict, path) -> Path:
    path = Path(path)
    path.write_text(json.dumps(doc))
    return path


def joint_limits(doc: dict) -> np.ndarray:
    """(D, 2) position limits of the actuated joints in declaration order."""
    rows = [j["limits"]["position"] for j in doc["joints"] if j["type"] != "fixed"]
    return np.asarray(rows, dtype=np.float64)


def random_configs(doc: dict, n: int, seed: int, shrink: float = 0.9) -> np.ndarray:
    """Configurations uniform within ``shrink`` x the joint limits."""
    lim = joint_limits(doc)
    rng = np.random.default_rng(seed)
    return rng.uniform(shrink * lim[:, 0], shrink * lim[:, 1], size=(n, len(lim)))


def smooth_trajectory(doc: dict, n: int, seed: int, shrink: float = 0.9) -> np.ndarray:
    """A time-parameterised path between two random configurations (config 5)."""
    lim = joint_limits(doc)
    rng = np.random.default_rng(seed)
    a = rng.uniform(shrink * lim[:, 0], shrink * lim[:, 1])
    b = rng.uniform(shrink * lim[:, 0], shrink * lim[:, 1])
    s = 0.5 - 0.5 * np.cos(np.linspace(0.0, np.pi, n))
    return a[None] + s[:, None] * (b - a)[None]


def human_cloud(n: int, seed: int, center=HUMAN_CENTER, sigma=HUMAN_SIGMA,
                clutter: float = 0.1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    n_clutter = int(round(clutter * n))
    blob = rng.normal(center, sigma, size=(n - n_clutter, 3))
    junk = rng.uniform(-1.0, 1.0, size=(n_clutter, 3))
    return np.concatenate([blob, junk], axis=0)


def crowd_cloud(n_humans: int, per_human: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-0.7, 0.7, size=(n_humans, 3))
    parts = [rng.normal(c, HUMAN_SIGMA, size=(per_human, 3)) for c in centers]
    return np.concatenate(parts, axis=0)


def far_crowd_cloud(n_points: int, seed: int) -> np.ndarray:
    """Config-4 robustness variant: the crowd's points packed into the eight
    corners of the grid (|x|, |y|, |z| in [0.8, 1)), out of most windows' reach."""
    rng = np.random.default_rng(seed)
    corner = rng.choice([-1.0, 1.0], size=(n_points, 3))
    return corner * rng.uniform(0.8, 1.0, size=(n_points, 3))


def sparse_cloud(n_points: int, seed: int) -> np.ndarray:
    """Config-4 robustness variant: a few uniform points over the grid (most windows empty or nearly)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n_points, 3))


def moving_human_frames(n_frames: int = 100, n_points: int = 30_000, seed: int = 0,
                        start_x: float = 1.4, speed: float = 1.6, dt: float = 0.008):
    """[(timestamp_ms, points)] for a blob approaching the base along -x."""
    rng = np.random.default_rng(seed)
    base = rng.normal(0.0, HUMAN_SIGMA, size=(n_points, 3))
    frames = []
    for k in range(n_frames):
        t = k * dt
        center = np.float64([start_x - speed * t, HUMAN_CENTER[1], HUMAN_CENTER[2]])
        jitter = rng.normal(0.0, 0.002, size=(n_points, 3))
        frames.append((1000.0 * t, base + center + jitter))
    return frames


@dataclass(frozen=True)
class ConfigShape:
    """One of BASELINE.json's configurations, restated as numbers."""

    name: str
    robot: dict
    n_waypoints: int
    n_points: int
    grid_extent: float = 1.0
    grid_res: float = 0.04
    link_extent: float = 0.32
    link_res: float = 0.02
    cloud: str = "human"


CONFIG1 = ConfigShape("config1_cpu_ref", ARM6G, 500, 10_000, link_res=0.02)
CONFIG2 = ConfigShape("config2_realtime", ARM6G, 500, 100_000, link_res=0.01)
CONFIG4 = ConfigShape("config4_throughput", ARM7G, 65_536, 1_000_000, link_res=0.01,
                      cloud="crowd")
CONFIG5 = ConfigShape("config5_dynamic", ARM6G, 500, 30_000, link_res=0.01, cloud="moving")


def cloud_for(shape: ConfigShape, seed: int) -> np.ndarray:
    if shape.cloud == "human":
        return human_cloud(shape.n_points, seed)
    if shape.cloud == "crowd":
        return crowd_cloud(10, shape.n_points // 10, seed)
    raise ValueError(f"no single cloud for {shape.cloud}")
