"""CPU: the C restatement (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py). This pins the checker used by
the GPU parity tests when /root/reference is absent."""
import os

import numpy as np
import pytest

from oracle.pyoracle import Scene

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cvp_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def small_scene(g):
    return Scene((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, g["small_views"])


def test_trajectory_and_rng_bitwise(gold, restatement):
    v = restatement.circular_trajectory(40.0, 70.0, 4, 360.0, 32, 32, 1.0, 1.0)
    assert np.array_equal(v, gold["small_views"])
    v = restatement.circular_trajectory(749.0, 1198.0, 36, 200.0, 480, 616, 0.154, 0.154)
    assert np.array_equal(v, gold["carm_views"])
    assert np.array_equal(restatement.fill_uniform01(16, 7), gold["rng_seed7_first16"])


@pytest.mark.parametrize("key", ["0000", "0001", "0100", "0101", "1000", "1001", "1100", "1101"])
def test_cvp_double_all_combos(gold, restatement, key):
    opts = tuple(int(c) for c in key)
    sc = small_scene(gold)
    p = restatement.project_cvp(sc, gold["small_x"], opts)
    bp = restatement.backproject_cvp(sc, gold["small_b"], opts)
    ref_p, ref_bp = gold[f"P_{key}"], gold[f"BP_{key}"]
    assert np.abs(p - ref_p).max() <= 1e-10 * np.abs(ref_p).max()
    assert np.abs(bp - ref_bp).max() <= 1e-10 * np.abs(ref_bp).max()


def test_cvp_single(gold, restatement):
    sc = small_scene(gold)
    p = restatement.project_cvp(sc, gold["small_x"], (1, 1, 1, 1))
    bp = restatement.backproject_cvp(sc, gold["small_b"], (1, 1, 1, 1))
    # both sides are float32 kernels; they differ only in rounding/FMA order
    assert np.linalg.norm(p - gold["P_1111"]) <= 1e-5 * np.linalg.norm(gold["P_1111"])
    assert np.linalg.norm(bp - gold["BP_1111"]) <= 1e-5 * np.linalg.norm(gold["BP_1111"])


def test_cut_records(gold, restatement):
    cviews = gold["carm_views"]
    sc = Scene((64, 64, 64), (0.72, 0.72, 0.72), 480, 616, 0.154, 0.154, cviews)
    recs = gold["carm_records"]
    for t in np.unique(recs[:, 0]):
        rows = recs[recs[:, 0] == t]
        _, i, j, k, v, s_, e, p, r = (int(x) for x in rows[0, :9])
        rr, rc, rv, ri = restatement.collect_cut_records(sc, cviews[v], (s_, e, p, r), i, j, k)
        assert len(rr) == len(rows)
        np.testing.assert_array_equal(rr, rows[:, 9].astype(int))
        np.testing.assert_array_equal(rc, rows[:, 10].astype(int))
        np.testing.assert_allclose(rv, rows[:, 11], rtol=1e-9, atol=1e-15)
        np.testing.assert_allclose(ri, rows[:, 12], rtol=1e-12)
        # conservation (test_cvp.cpp:410-432)
        assert abs(rv.sum() - 0.72 ** 3) <= 1e-9


def test_pixel_scales(gold, restatement):
    cviews = gold["carm_views"]
    sc = Scene((64, 64, 64), (0.72, 0.72, 0.72), 480, 616, 0.154, 0.154, cviews)
    for (m, n), ex, co in zip(gold["carm_scale_px"], gold["carm_scale_exact"],
                              gold["carm_scale_cos"]):
        # exact form: 2*pi - sum(acos) cancels ~1e-7 relative at 0.154 mm pixels (cvp.cpp:580-598)
        assert restatement.pixel_scale(sc, cviews[3], 1, int(m), int(n)) == pytest.approx(ex, rel=1e-6)
        assert restatement.pixel_scale(sc, cviews[3], 0, int(m), int(n)) == pytest.approx(co, rel=1e-13)


@pytest.mark.parametrize("K", [1, 2])
def test_siddon(gold, restatement, K):
    sc = small_scene(gold)
    p = restatement.project_siddon(sc, gold["small_x"], K)
    bp = restatement.backproject_siddon(sc, gold["small_b"], K)
    assert np.abs(p - gold[f"SID_P_{K}"]).max() <= 1e-12 * np.abs(gold[f"SID_P_{K}"]).max()
    assert np.abs(bp - gold[f"SID_BP_{K}"]).max() <= 1e-12 * np.abs(gold[f"SID_BP_{K}"]).max()


def test_dot_kahan_and_reference_adjointness(gold, restatement):
    # the reference's own adjoint test result is at the 1e-12 level (test_cvp.cpp:349-373)
    assert float(gold["adjoint_cvp_seed1"]) < 1e-12
    assert float(gold["adjoint_sid2_seed1"]) < 1e-12
    import ctypes as C
    import math
    a = gold["small_x"]
    f = restatement.lib.orc_dot_kahan
    f.restype = C.c_double
    f.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t]
    pa = a.ctypes.data_as(C.POINTER(C.c_double))
    assert f(pa, pa, a.size) == pytest.approx(math.fsum(a * a), rel=1e-15)


def test_reference_matches_golden_when_present(gold, reference):
    sc = small_scene(gold)
    p = reference.project_cvp(sc, gold["small_x"], (1, 1, 0, 1), threads=1)
    assert np.array_equal(p, gold["P_1101"])
