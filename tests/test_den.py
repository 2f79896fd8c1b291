"""CPU (+1 GPU case): DEN I/O (den.cpp), restated from the reference's
test_den.cpp, plus the zero-conversion device loader."""
import os

import numpy as np
import pytest

import paper_2110_09841_b200 as cb
from paper_2110_09841_b200 import den


def test_volume_roundtrip(tmp_path):
    geom = cb.VolumeGeometry.make((2, 3, 4), (0.5, 0.25, 1.0))
    vol = cb.AttenuationVolume(geom, np.arange(24, dtype=np.float64))
    d = den.to_den(vol)
    assert (d.dim_y, d.dim_x, d.dim_z) == (3, 2, 4)
    assert np.array_equal(d.values, np.arange(24, dtype=np.float32))
    p = tmp_path / "v.den"
    den.den_write(p, d)
    back = den.volume_from_den(den.den_read(p), (0.5, 0.25, 1.0))
    assert back.geom == geom and np.array_equal(back.values, vol.values)
    q = tmp_path / "w.den"
    den.den_write(q, den.den_read(p))
    assert open(p, "rb").read() == open(q, "rb").read()
    assert os.path.getsize(p) == 6 + 4 * 24


def test_stack_roundtrip(tmp_path):
    det = cb.DetectorGeometry.make(3, 5, 0.2, 0.3)
    proj = cb.ProjectionStack(det, 2, np.linspace(-1, 1, 30))
    d = den.to_den(proj)
    assert (d.dim_y, d.dim_x, d.dim_z) == (3, 5, 2)
    den.den_write(tmp_path / "s.den", d)
    back = den.stack_from_den(den.den_read(tmp_path / "s.den"), 0.2, 0.3)
    assert back.det == det and back.n_views == 2
    assert np.array_equal(back.values, proj.values.astype(np.float32).astype(np.float64))


def test_full_scale_header_size_message(tmp_path):
    p = tmp_path / "big.den"
    with open(p, "wb") as f:
        f.write(np.array([512, 512, 720], dtype="<u2").tobytes())
        f.write(np.zeros(1, dtype="<f4").tobytes())
    with pytest.raises(RuntimeError, match="754974726"):
        den.den_read(p)


def test_malformed_files(tmp_path):
    empty = tmp_path / "e.den"
    empty.write_bytes(b"")
    with pytest.raises(RuntimeError):
        den.den_read(empty)
    with pytest.raises(RuntimeError):
        den.den_read(tmp_path / "missing.den")
    zero = tmp_path / "z.den"
    zero.write_bytes(np.array([0, 4, 4], dtype="<u2").tobytes())
    with pytest.raises(RuntimeError):
        den.den_read(zero)


def test_write_validation_and_cap(tmp_path):
    with pytest.raises(RuntimeError):
        den.den_write(tmp_path / "b.den", den.DenFile(2, 2, 1, np.zeros(3, np.float32)))
    with pytest.raises(RuntimeError):
        den.den_write(tmp_path / "b.den", den.DenFile(2, 2, 0, np.zeros(0, np.float32)))
    geom = cb.VolumeGeometry.make((70000, 1, 1), (0.01, 1.0, 1.0))
    with pytest.raises(RuntimeError):
        den.to_den(cb.AttenuationVolume.zeros(geom))


@pytest.mark.gpu
def test_device_loader_matches_layout(tmp_path):
    import torch
    geom = cb.VolumeGeometry.make((4, 3, 2), (1.0, 1.0, 1.0))
    vol = cb.AttenuationVolume(geom, np.arange(24, dtype=np.float64))
    den.den_write(tmp_path / "v.den", den.to_den(vol))
    t = den.den_read_device(tmp_path / "v.den")
    torch.cuda.synchronize()
    assert t.shape == geom.shape() and t.is_cuda
    assert torch.equal(t.cpu().view(-1), torch.arange(24, dtype=torch.float32))
    den.den_write_device(tmp_path / "w.den", t)
    assert open(tmp_path / "v.den", "rb").read() == open(tmp_path / "w.den", "rb").read()


# ---- byte-exact parity with the reference's own den.cpp (oracle/_ref) -------

def _ref_lib():
    import ctypes as C
    from oracle import pyoracle
    if not pyoracle.reference_available():
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(pyoracle.REFERENCE_SO)
    lib.ref_den_write.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
    lib.ref_den_read.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_float), C.c_size_t]
    lib.ref_den_write_volume.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
    lib.ref_last_error.restype = C.c_char_p
    return lib


def test_den_bytes_match_the_reference_writer(tmp_path):
    """den.py and the reference's den_write produce identical files; each
    reads the other's file back to the same values (den.cpp:27-68)."""
    import ctypes as C
    lib = _ref_lib()
    rng = np.random.default_rng(5)
    vals = (rng.standard_normal(7 * 5 * 3) * 1e3).astype(np.float32)
    vals[:4] = [0.0, -0.0, np.inf, np.nan]
    ours, theirs = tmp_path / "ours.den", tmp_path / "theirs.den"
    den.den_write(ours, den.DenFile(7, 5, 3, vals))
    assert lib.ref_den_write(str(theirs).encode(), 7, 5, 3,
                             vals.ctypes.data_as(C.POINTER(C.c_float))) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    dims = (C.c_int * 3)()
    back = np.zeros(vals.size, dtype=np.float32)
    assert lib.ref_den_read(str(ours).encode(), dims, back.ctypes.data_as(C.POINTER(C.c_float)),
                            back.size) == 0
    assert tuple(dims) == (7, 5, 3)
    assert back.tobytes() == vals.tobytes()
    d = den.den_read(theirs)
    assert (d.dim_y, d.dim_x, d.dim_z) == (7, 5, 3) and d.values.tobytes() == vals.tobytes()


def test_den_volume_mapping_matches_the_reference(tmp_path):
    """to_den of a float64 volume (N2, N1, N3 header, float32 payload):
    byte-identical to the reference's to_den + den_write (den.cpp:70-79)."""
    import ctypes as C
    lib = _ref_lib()
    geom = cb.VolumeGeometry.make((6, 4, 3), (0.5, 0.25, 1.0))
    x = cb.fill_uniform01(geom.voxel_count(), 11) * 3.0 - 1.0
    ours, theirs = tmp_path / "v_ours.den", tmp_path / "v_theirs.den"
    den.den_write(ours, den.to_den(cb.AttenuationVolume(geom, x)))
    counts = (C.c_int * 3)(6, 4, 3)
    voxel = (C.c_double * 3)(0.5, 0.25, 1.0)
    assert lib.ref_den_write_volume(str(theirs).encode(), counts, voxel,
                                    x.ctypes.data_as(C.POINTER(C.c_double))) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_den_reference_rejects_what_den_py_rejects(tmp_path):
    """Malformed files: both sides refuse (size mismatch, truncated header)."""
    import ctypes as C
    lib = _ref_lib()
    bad = tmp_path / "bad.den"
    bad.write_bytes(np.array([2, 2, 2], dtype="<u2").tobytes() + b"\0" * 8)
    dims = (C.c_int * 3)()
    buf = np.zeros(8, dtype=np.float32)
    assert lib.ref_den_read(str(bad).encode(), dims, buf.ctypes.data_as(C.POINTER(C.c_float)), 8) != 0
    with pytest.raises(cb.CvpbRuntimeError):
        den.den_read(bad)
    short = tmp_path / "short.den"
    short.write_bytes(b"\1\0")
    assert lib.ref_den_read(str(short).encode(), dims, buf.ctypes.data_as(C.POINTER(C.c_float)), 8) != 0
    with pytest.raises(cb.CvpbRuntimeError):
        den.den_read(short)
