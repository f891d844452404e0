"""CPU checks of the boundary: libholo.so loads and exports every symbol include/holo.h
declares (no compute calls without a GPU); host-side argument validation."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "holo.h")


def declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(holo_[a-z0-9_]+)\s*\(", txt)) - {"holo_status"})


def test_header_declares_the_north_star_entry_points():
    d = declared()
    for name in ["holo_fwd", "holo_adj", "holo_grad", "holo_cg_step", "holo_plan_create", "holo_q_dots",
                 "holo_grad_ref"]:
        assert name in d


def test_library_exports_every_declared_symbol():
    import paper_2407_20304_b200 as hb
    out = subprocess.run(["nm", "-D", "--defined-only", hb.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (holo_[a-z0-9_]+)", out))
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    assert set(hb.EXPORTED) <= exported


def test_library_is_sm100a():
    import paper_2407_20304_b200 as hb
    out = subprocess.run(["cuobjdump", "--list-elf", hb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_plan_create_validates_geometry_without_gpu():
    """Invalid geometry is rejected on the host before any CUDA call (HOLO_EINVAL / HOLO_EUNSUPPORTED)."""
    import ctypes
    import paper_2407_20304_b200 as hb
    g = hb.HoloGeometry()
    g.n, g.npad, g.nz, g.n_angles, g.angle_batch = 64, 128, 2, 1, 1
    g.wavelength, g.focus_to_detector, g.detector_pixel = 3.7e-11, 1.208, 3e-6
    g.z1[0], g.z1[1] = 5e-3, 4e-3  # not increasing
    h = ctypes.c_void_p()
    assert hb._lib.holo_plan_create(ctypes.byref(h), ctypes.byref(g), 0, None) == hb.HOLO_EINVAL
    g.z1[1] = 6e-3
    g.npad = 96  # not a power of two
    assert hb._lib.holo_plan_create(ctypes.byref(h), ctypes.byref(g), 0, None) == hb.HOLO_EUNSUPPORTED
    g.npad, g.n = 128, 63  # odd n
    assert hb._lib.holo_plan_create(ctypes.byref(h), ctypes.byref(g), 0, None) == hb.HOLO_EINVAL
    g.n, g.wavelength = 64, -1.0
    assert hb._lib.holo_plan_create(ctypes.byref(h), ctypes.byref(g), 0, None) == hb.HOLO_EINVAL


def test_binding_refuses_cpu_tensors():
    import torch
    import paper_2407_20304_b200 as hb
    with pytest.raises(ValueError):
        hb._ptr(torch.zeros(4, dtype=torch.complex64), torch.complex64, 4, "x")
