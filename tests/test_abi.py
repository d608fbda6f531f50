"""CPU: the C-ABI library builds, loads and exports exactly what include/kct.h
declares; argument validation (ConfigError) happens before any device work."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2509_08574_b200 as k

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kct.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kct_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_header():
    lib = k.load_library()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(k._SIGS), "python bindings must cover the header exactly"
    assert lib.kct_abi_version() == 4


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {k.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def _create(grid, geom):
    lib = k.load_library()
    h = C.c_void_p()
    g, ge = grid._c(), geom._c()
    return lib.kct_projector_create(C.byref(g), C.byref(ge), -1, C.byref(h))


@pytest.mark.parametrize("mut", ["dims", "spacing", "dsd", "pixels", "pitch", "angles", "inside"])
def test_config_errors(mut):
    """types.hpp:72-77, :152-160; projector.hpp:162-168 (test_projector.cpp:113-120)."""
    grid = k.GridSpec((8, 8, 8), (1.0, 1.0, 1.0))
    geom = k.ConeBeamGeometry(40.0, 90.0, 10, 9, 1.6, 1.9, k.uniform_angles(4))
    if mut == "dims":
        grid = k.GridSpec((0, 8, 8))
    elif mut == "spacing":
        grid = k.GridSpec((8, 8, 8), (1.0, -1.0, 1.0))
    elif mut == "dsd":
        geom.dsd = 30.0
    elif mut == "pixels":
        geom.nu = 0
    elif mut == "pitch":
        geom.pv = 0.0
    elif mut == "angles":
        geom.angles = np.zeros(0)
    elif mut == "inside":
        grid = k.GridSpec((32, 32, 32), (10.0, 10.0, 10.0))
    assert _create(grid, geom) == 2
    assert k.load_library().kct_last_error()


def test_python_raises_config_error():
    with pytest.raises(k.ConfigError):
        k.ConeBeamProjector(k.GridSpec((32, 32, 32), (10.0, 10.0, 10.0)),
                            k.ConeBeamGeometry(40.0, 90.0, 4, 4, 1.0, 1.0, k.uniform_angles(4)))


def test_resolve_tau_host():
    """test_recon.cpp:72-86 through the C ABI."""
    assert k.resolve_tau(0.5) == 0.5
    assert k.resolve_tau(0.0) == 1e-4
    assert k.resolve_tau(0.0, [0.25, 1.0, 2.25]) == pytest.approx(2e-4, rel=1e-12)
    assert k.resolve_tau(0.0, [0.7] * 10) == 1e-4
    assert k.resolve_tau(0.0, [0.0, 1e-6]) == pytest.approx(1e-8)


def test_subsample():
    """test_projector.cpp:122-141."""
    assert k.subsample_indices(10, 4) == [0, 2, 5, 7]
    assert k.subsample_indices(7, 1) == [0]
    with pytest.raises(k.ConfigError):
        k.subsample_indices(5, 6)
    g = k.ConeBeamGeometry(40.0, 90.0, 3, 2, 1.0, 1.0, k.uniform_angles(10))
    full = k.ProjectionSet(g, np.arange(g.ray_count(), dtype=np.float32))
    sub = k.subsample_angles(full, 4)
    assert sub.geometry.n_angles() == 4
    np.testing.assert_array_equal(sub.geometry.angles, g.angles[[0, 2, 5, 7]])
    np.testing.assert_array_equal(sub.data.reshape(4, 6)[1], full.data.reshape(10, 6)[2])
