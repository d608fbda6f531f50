"""On-disk exchange format of the reference (io.hpp:30-163): raw little-endian
float32 next to a "<name>.meta.json" sidecar — volumes x-fastest, projection
stacks u-fastest.  Files written here are read by the reference CLI
(`kryct metrics`, `prior.kind = "file"`) and vice versa; a float32 round trip
is byte-stable.  Host-side only (numpy); device arrays are converted by the
callers (``ConeBeamProjector.volume_from_native`` / ``proj_from_native``).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

from . import ConeBeamGeometry, ConfigError, GridSpec, ProjectionSet

if sys.byteorder != "little":  # io.hpp:25-26
    raise ImportError("raw volume io assumes a little-endian host")


def _pair(stem) -> tuple[str, str]:
    """io.hpp:57-67: "<dir>/name" or "<dir>/name.raw" -> (raw, meta)."""
    stem = os.fspath(stem)
    if stem.endswith(".raw"):
        stem = stem[:-4]
    return stem + ".raw", stem + ".meta.json"


def _load_meta(path: str) -> dict:
    try:
        with open(path) as f:
            return json.load(f)
    except OSError as e:
        raise ConfigError(f"cannot open metadata: {path}") from e
    except json.JSONDecodeError as e:
        raise ConfigError(f"bad metadata in {path}: {e}") from e


def _read_raw(path: str, count: int) -> np.ndarray:
    try:
        data = np.fromfile(path, dtype="<f4", count=count)
    except OSError as e:
        raise ConfigError(f"cannot open for reading: {path}") from e
    if data.size != count:
        raise ConfigError(f"raw file shorter than its metadata claims: {path}")
    return data


def _check_finite(a: np.ndarray, what: str) -> None:
    if not np.all(np.isfinite(a)):
        raise ConfigError(f"{what} contains non-finite values")


def write_volume(stem, grid: GridSpec, data) -> None:
    """io.hpp:78-93."""
    a = np.ascontiguousarray(np.asarray(data, dtype="<f4").reshape(-1))
    if a.size != grid.count():
        raise ConfigError("volume data length does not match dims")
    _check_finite(a, "volume")
    raw, meta = _pair(stem)
    a.tofile(raw)
    with open(meta, "w") as f:
        json.dump({"type": "volume", "dtype": "float32", "dims": list(grid.dims),
                   "spacing": list(grid.spacing), "origin": list(grid.origin),
                   "order": "x-fastest"}, f, indent=2)
        f.write("\n")


def read_volume(stem) -> tuple[GridSpec, np.ndarray]:
    """io.hpp:95-115."""
    raw, meta = _pair(stem)
    j = _load_meta(meta)
    try:
        if j["type"] != "volume":
            raise ConfigError(f"{meta} does not describe a volume")
        grid = GridSpec(tuple(int(v) for v in j["dims"]), tuple(float(v) for v in j["spacing"]),
                        tuple(float(v) for v in j["origin"]))
    except (KeyError, IndexError, TypeError, ValueError) as e:
        raise ConfigError(f"bad metadata in {meta}: {e}") from e
    data = _read_raw(raw, grid.count())
    _check_finite(data, "volume")
    return grid, data


def write_projections(stem, proj: ProjectionSet) -> None:
    """io.hpp:117-137."""
    g = proj.geometry
    a = np.ascontiguousarray(np.asarray(proj.data, dtype="<f4").reshape(-1))
    if a.size != g.ray_count():
        raise ConfigError("projection data length does not match geometry")
    _check_finite(a, "projections")
    raw, meta = _pair(stem)
    a.tofile(raw)
    with open(meta, "w") as f:
        json.dump({"type": "projections", "dtype": "float32", "order": "u-fastest",
                   "geometry": {"dso": g.dso, "dsd": g.dsd,
                                "detector": {"nu": g.nu, "nv": g.nv, "pu": g.pu, "pv": g.pv},
                                "offsets": [g.offset_u, g.offset_v],
                                "angles": [float(t) for t in g.angles]}}, f, indent=2)
        f.write("\n")


def read_projections(stem) -> ProjectionSet:
    """io.hpp:139-163."""
    raw, meta = _pair(stem)
    j = _load_meta(meta)
    try:
        if j["type"] != "projections":
            raise ConfigError(f"{meta} does not describe projections")
        jg = j["geometry"]
        d = jg["detector"]
        g = ConeBeamGeometry(float(jg["dso"]), float(jg["dsd"]), int(d["nu"]), int(d["nv"]),
                             float(d["pu"]), float(d["pv"]), np.asarray(jg["angles"], dtype=float),
                             float(jg["offsets"][0]), float(jg["offsets"][1]))
    except (KeyError, IndexError, TypeError, ValueError) as e:
        raise ConfigError(f"bad metadata in {meta}: {e}") from e
    data = _read_raw(raw, g.ray_count())
    _check_finite(data, "projections")
    return ProjectionSet(g, data)
