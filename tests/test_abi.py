"""CPU: the C-ABI library loads, exports every symbol include/cvpb200.h
declares, binds them all in the Python layer, and refuses to compute without
a GPU (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cvpb200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cvpb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_operator_surface():
    names = declared()
    for must in ["cvpb_project_cvp", "cvpb_backproject_cvp", "cvpb_project_cvp_host",
                 "cvpb_backproject_cvp_host", "cvpb_project_siddon", "cvpb_backproject_siddon",
                 "cvpb_project_tt", "cvpb_backproject_tt", "cvpb_cgls", "cvpb_vec_dot",
                 "cvpb_set_geometry", "cvpb_make_circular_trajectory",
                 "cvpb_view_from_standard_matrix", "cvpb_collect_cut_records"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2110_09841_b200 import _native
    lib = C.CDLL(_native.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (cvpb_[a-z0-9_]+)", out))
    assert set(declared()) <= exported


def test_python_binding_covers_the_header():
    from paper_2110_09841_b200 import _native
    assert set(declared()) == set(_native.SIGNATURES)
    _native.lib()  # binds every signature


def test_abi_version_and_no_cpu_fallback():
    import torch
    from paper_2110_09841_b200 import _native
    L = _native.lib()
    assert L.cvpb_abi_version() == 3
    n = C.c_int()
    assert L.cvpb_device_count(C.byref(n)) == 0
    if torch.cuda.is_available():
        pytest.skip("GPU present: the no-device path is not reachable")
    h = C.c_void_p()
    assert L.cvpb_context_create(0, C.byref(h)) == _native.NO_DEVICE
    assert b"no CPU fallback" in L.cvpb_last_error()
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(8, 8, 1.0, 1.0)
    views = cb.make_circular_trajectory(40.0, 70.0, 2, 360.0, det)
    with pytest.raises(cb.NoDevice):
        cb.DeviceScene(cb.VolumeGeometry.make((4, 4, 4), (1, 1, 1)), det, views)
