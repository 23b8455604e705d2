"""Streaming file formats (query.py:313-355): frame files,
manifests and the distance CSV — host plumbing, CPU only."""

import struct

import numpy as np
import pytest

from paper_2309_12543_b200 import query as Q
from paper_2309_12543_b200.errors import ValidationError


def test_frame_bytes_and_round_trip(tmp_path):
    pts = np.float64([[0.1, -0.2, 0.3], [1.5, 2.5, -3.5]])
    f = tmp_path / "f.bin"
    Q.write_pointcloud_frame(f, pts)
    raw = f.read_bytes()
    assert raw[:4] == struct.pack("<I", 2) and len(raw) == 4 + 2 * 12
    assert np.array_equal(np.frombuffer(raw[4:], "<f4").reshape(2, 3), pts.astype(np.float32))
    back = Q.read_pointcloud_frame(f)
    assert back.dtype == np.float64 and np.array_equal(back, pts.astype(np.float32).astype(np.float64))
    f.write_bytes(raw[:-1])
    with pytest.raises(ValidationError):
        Q.read_pointcloud_frame(f)
    Q.write_pointcloud_frame(f, np.zeros((0, 3)))
    assert Q.read_pointcloud_frame(f).shape == (0, 3)


def test_manifest_and_frames(tmp_path):
    for i in range(3):
        Q.write_pointcloud_frame(tmp_path / f"{i}.bin", np.full((i + 1, 3), float(i)))
    (tmp_path / "m.txt").write_text("# t_ms file\n0 0.bin\n\n8.0 1.bin\n16.5   2.bin\n")
    man = Q.read_cloud_manifest(tmp_path / "m.txt")
    assert [s for s, _ in man] == [0.0, 8.0, 16.5] and man[2][1] == tmp_path / "2.bin"
    frames = list(Q.iter_cloud_frames(tmp_path / "m.txt"))
    assert [len(p) for _, p in frames] == [1, 2, 3] and frames[2][1][0, 0] == 2.0


def test_distance_csv(tmp_path):
    f = tmp_path / "d.csv"
    Q.write_distance_csv(f, [(0.0, np.float32([0.1, -0.25])), (8.25, np.float32([0.3, 0.0]))], 2)
    assert f.read_text().splitlines() == ["timestamp_ms,d_0,d_1", "0.000,0.100000,-0.250000",
                                          "8.250,0.300000,0.000000"]


def test_link_sdf_file_round_trip(tmp_path):
    """LSDF cache file (grids.py:218-257): header + x-fastest f32 values."""
    from paper_2309_12543_b200 import grids as G

    vals = np.arange(4 * 5 * 6, dtype=np.float32).reshape(4, 5, 6) / 7.0
    sdf = G.LinkSdf(extent=[0.2, 0.25, 0.3], resolution=0.1, values=vals, link_id=3)
    f = tmp_path / "l.lsdf"
    G.write_link_sdf(f, sdf)
    raw = f.read_bytes()
    head = struct.calcsize(G._HEADER)
    assert raw[:4] == G.LSDF_MAGIC and len(raw) == head + 4 * vals.size
    assert np.array_equal(np.frombuffer(raw[head:], "<f4"), vals.ravel(order="F"))
    back = G.read_link_sdf(f)
    assert back.link_id == 3 and np.array_equal(back.values, vals)
    # the header stores extent and resolution as f32 (the reference's format)
    assert np.array_equal(back.extent, sdf.extent.astype(np.float32))
    assert np.array_equal(back.resolution, sdf.resolution.astype(np.float32))
    f.write_bytes(raw[:-4])
    with pytest.raises(ValidationError):
        G.read_link_sdf(f)
    f.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValidationError):
        G.read_link_sdf(f)


def test_tmlp_file_round_trip(tmp_path):
    """TMLP weights file (approx.py:132-158)."""
    from paper_2309_12543_b200.approx import TMLP_MAGIC, TinyMlp

    m = TinyMlp.random(10, hidden=20, seed=2)
    f = tmp_path / "m.tmlp"
    m.save(f)
    raw = f.read_bytes()
    assert raw[:4] == TMLP_MAGIC and struct.unpack("<III", raw[4:16])[1:] == (20, 10)
    back = TinyMlp.load(f)
    for k in ("w1", "b1", "w2", "b2"):
        assert np.array_equal(getattr(back, k), getattr(m, k))
    f.write_bytes(raw[:-1])
    with pytest.raises(ValidationError):
        TinyMlp.load(f)
