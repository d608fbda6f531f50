"""CPU: raw-f32 + meta.json exchange format (io.hpp:30-163)."""
import json

import numpy as np
import pytest

import paper_2509_08574_b200 as k
from paper_2509_08574_b200 import io


def test_volume_round_trip(tmp_path):
    grid = k.GridSpec((5, 4, 3), (1.0, 1.1, 0.9))
    data = np.random.default_rng(0).standard_normal(grid.count()).astype(np.float32)
    io.write_volume(tmp_path / "vol", grid, data)
    meta = json.load(open(tmp_path / "vol.meta.json"))
    assert meta["type"] == "volume" and meta["order"] == "x-fastest"
    assert meta["dims"] == [5, 4, 3] and meta["dtype"] == "float32"
    g2, d2 = io.read_volume(tmp_path / "vol.raw")
    assert g2 == grid
    assert d2.tobytes() == data.tobytes()  # byte-stable
    assert (tmp_path / "vol.raw").stat().st_size == 4 * grid.count()


def test_projection_round_trip(tmp_path):
    geom = k.ConeBeamGeometry(40.0, 90.0, 10, 9, 1.6, 1.9, k.uniform_angles(8), 0.7, -0.5)
    p = k.ProjectionSet(geom, np.arange(geom.ray_count(), dtype=np.float32))
    io.write_projections(tmp_path / "p", p)
    meta = json.load(open(tmp_path / "p.meta.json"))
    assert meta["geometry"]["detector"] == {"nu": 10, "nv": 9, "pu": 1.6, "pv": 1.9}
    assert meta["geometry"]["offsets"] == [0.7, -0.5]
    q = io.read_projections(tmp_path / "p")
    np.testing.assert_array_equal(q.geometry.angles, geom.angles)
    assert q.data.tobytes() == p.data.tobytes()


def test_errors(tmp_path):
    grid = k.GridSpec((2, 2, 2))
    with pytest.raises(k.ConfigError):
        io.write_volume(tmp_path / "v", grid, np.zeros(7))
    with pytest.raises(k.ConfigError):
        io.write_volume(tmp_path / "v", grid, np.full(8, np.nan))
    io.write_volume(tmp_path / "v", grid, np.zeros(8))
    (tmp_path / "v.raw").write_bytes(b"\0" * 12)
    with pytest.raises(k.ConfigError):
        io.read_volume(tmp_path / "v")
    with pytest.raises(k.ConfigError):
        io.read_projections(tmp_path / "v")
    with pytest.raises(k.ConfigError):
        io.read_volume(tmp_path / "missing")
