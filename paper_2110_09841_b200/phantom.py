"""Deterministic 3D Shepp–Logan phantom (host-side input generator).

Kak & Slaney's ellipsoid set with Toft's "modified" intensities, normalised
to [-1, 1]^3 and sampled at voxel centres of a VolumeGeometry. The
reference ships no phantom generator; BASELINE.json configs[0]
asks for one, so both the GPU path and the CPU oracle read the same array
produced here.
"""
from __future__ import annotations

import numpy as np

from .geometry import VolumeGeometry

#        A      a      b      c      x0      y0      z0    phi  theta  psi
_ELLIPSOIDS = np.array([
    [1.0, .6900, .920, .810, 0.00, 0.000, 0.00, 0.0, 0.0, 0.0],
    [-.8, .6624, .874, .780, 0.00, -.0184, 0.00, 0.0, 0.0, 0.0],
    [-.2, .1100, .310, .220, 0.22, 0.000, 0.00, -18., 0.0, 10.],
    [-.2, .1600, .410, .280, -.22, 0.000, 0.00, 18.0, 0.0, 10.],
    [0.1, .2100, .250, .410, 0.00, 0.350, -.15, 0.0, 0.0, 0.0],
    [0.1, .0460, .046, .050, 0.00, 0.100, 0.25, 0.0, 0.0, 0.0],
    [0.1, .0460, .046, .050, 0.00, -.100, 0.25, 0.0, 0.0, 0.0],
    [0.1, .0460, .023, .050, -.08, -.605, 0.00, 0.0, 0.0, 0.0],
    [0.1, .0230, .023, .020, 0.00, -.606, 0.00, 0.0, 0.0, 0.0],
    [0.1, .0230, .046, .020, 0.06, -.605, 0.00, 0.0, 0.0, 0.0],
])


def _euler(phi, theta, psi):
    cph, sph = np.cos(phi), np.sin(phi)
    cth, sth = np.cos(theta), np.sin(theta)
    cps, sps = np.cos(psi), np.sin(psi)
    return np.array([
        [cps * cph - cth * sph * sps, cps * sph + cth * cph * sps, sps * sth],
        [-sps * cph - cth * sph * cps, -sps * sph + cth * cph * cps, cps * sth],
        [sth * sph, -sth * cph, cth],
    ])


def shepp_logan_3d(geom: VolumeGeometry, scale: float = 1.0) -> np.ndarray:
    """float64 array in the reference volume layout (flat, i fastest); the
    phantom's unit cube is mapped onto the volume box."""
    n1, n2, n3 = geom.counts
    # normalised voxel-centre coordinates in [-1, 1]
    u = (np.arange(n1) + 0.5) / n1 * 2.0 - 1.0
    v = (np.arange(n2) + 0.5) / n2 * 2.0 - 1.0
    w = (np.arange(n3) + 0.5) / n3 * 2.0 - 1.0
    Z, Y, X = np.meshgrid(w, v, u, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()])
    out = np.zeros(pts.shape[1])
    for A, a, b, c, x0, y0, z0, phi, theta, psi in _ELLIPSOIDS:
        R = _euler(np.deg2rad(phi), np.deg2rad(theta), np.deg2rad(psi))
        q = R @ pts
        inside = ((q[0] - x0) ** 2 / a ** 2 + (q[1] - y0) ** 2 / b ** 2 +
                  (q[2] - z0) ** 2 / c ** 2) <= 1.0
        out[inside] += A
    return out * scale
