"""CPU: the SF-TT oracle (oracle/tt_oracle.c, float64 restatement of Long,
Fessler & Balter 2010) against the paper's own properties — known answers of
the separable-footprint model — before it is trusted as the GPU TT checker:

* the transaxial footprint of a voxel, summed over detector columns, is the
  trapezoid's area ((tau3 - tau0) + (tau2 - tau1)) / 2 (cell averages of a
  unit-height trapezoid integrate it exactly);
* the axial footprint likewise; their product with the amplitude is the
  voxel's whole contribution;
* the pair is an exact transpose (<Ax, y> = <x, A'y> to float64 rounding);
* linearity, and the A2 amplitude reduces to A1 on the central detector row.
"""
import numpy as np
import pytest

from oracle.pyoracle import Restatement, Scene


def _scene(n=8, rows=48, cols=48, px=1.0, sid=60.0, sdd=100.0, nv=4):
    r = Restatement()
    views = r.circular_trajectory(sid, sdd, nv, 360.0, rows, cols, px, px)
    return r, Scene((n, n, n), (1.0, 1.0, 1.0), rows, cols, px, px, views)


def test_tt_oracle_single_voxel_mass_is_trapezoid_area_times_amplitude():
    r, sc = _scene(n=1, nv=1)
    p = r.project_tt(sc, np.ones(1), amplitude=0)[0]
    # view 0: source on +x1 at (60, 0, 0); the voxel [-0.5, 0.5]^3 at the origin.
    # chi1 of the corners: pp1 + f * u / (b1 * depth), u = e_u . (x - s)
    v = sc.views[0]
    s, eu, ew, f, pp1, pp2 = v[0:3], v[3:6], v[9:12], v[12], v[13], v[14]
    tau, dep = [], []
    for dx in (-0.5, 0.5):
        for dy in (-0.5, 0.5):
            d = np.array([dx, dy, 0.0]) - s
            dep.append(ew @ d)
            tau.append(pp1 + f * (eu @ d) / dep[-1])
    tau = np.sort(tau)
    f1 = ((tau[3] - tau[0]) + (tau[2] - tau[1])) / 2
    t = np.sort([pp2 - z * f / dd for z in (-0.5, 0.5) for dd in (min(dep), max(dep))])
    f2 = ((t[3] - t[0]) + (t[2] - t[1])) / 2
    lphi = 1.0  # central ray along x1: l = a1 / |cos 0|
    assert p.sum() == pytest.approx(lphi * f1 * f2, rel=1e-12)


def test_tt_oracle_pair_is_an_exact_transpose_and_linear():
    r, sc = _scene(n=10, nv=5)
    rng = np.random.default_rng(3)
    x = rng.random(sc.nvox())
    y = rng.random(sc.npx())
    for amp in (0, 1):
        ax = r.project_tt(sc, x, amp).ravel()
        aty = r.backproject_tt(sc, y, amp).ravel()
        lhs, rhs = ax @ y, x @ aty
        assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), abs(rhs))
        assert np.allclose(r.project_tt(sc, 2.0 * x, amp).ravel(), 2.0 * ax, rtol=0, atol=1e-12 * ax.max())


def test_tt_oracle_amplitudes_agree_on_the_central_row():
    # a voxel on the central plane z = 0 projects onto row pp2: A1 = A2 there
    r, sc = _scene(n=1, rows=49, cols=48, nv=3)
    p1 = r.project_tt(sc, np.ones(1), 0)
    p2 = r.project_tt(sc, np.ones(1), 1)
    assert np.allclose(p1[:, 24, :], p2[:, 24, :], rtol=1e-12)
    # off the central row the A2 amplitude grows with the elevation
    assert (p2[:, 23, :] >= p1[:, 23, :] * (1 - 1e-12)).all()
