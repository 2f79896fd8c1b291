"""Generate tests/golden/cvp_golden.npz from the REFERENCE itself.

Runs the unmodified reference library (/root/reference/proj/src compiled by
oracle/Makefile into oracle/_ref/libcbct_ref.so) on small pinned scenes and
stores inputs + outputs. The fixtures pin the C restatement (oracle/) and the
device path when the reference is not present (e.g. on the GPU box).

    make -C oracle ref && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference, Scene  # noqa: E402


def main():
    R = Reference()
    out = {}
    # scene of test_cvp.cpp:349-373 with 4 views
    views = R.circular_trajectory(40.0, 70.0, 4, 360.0, 32, 32, 1.0, 1.0)
    sc = Scene((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, views)
    out["small_views"] = views
    x = R.fill_uniform01(16 ** 3, 3)
    b = R.fill_uniform01(32 * 32 * 4, 5)
    out["small_x"] = x
    out["small_b"] = b
    for s_ in (0, 1):
        for e in (0, 1):
            for r in (0, 1):
                for prec in (0, 1):
                    if prec == 1 and (s_, e, r) != (1, 1, 1):
                        continue
                    key = f"{s_}{e}{prec}{r}"
                    out[f"P_{key}"] = R.project_cvp(sc, x, (s_, e, prec, r), threads=1)
                    out[f"BP_{key}"] = R.backproject_cvp(sc, b, (s_, e, prec, r), threads=1)
    # C-arm geometry (fine pixels) trajectory + scales + cut records
    det = (480, 616, 0.154, 0.154)
    cviews = R.circular_trajectory(749.0, 1198.0, 36, 200.0, *det)
    out["carm_views"] = cviews
    csc = Scene((64, 64, 64), (0.72, 0.72, 0.72), *det, cviews)
    px = [(0, 0), (240, 308), (479, 615), (100, 500)]
    out["carm_scale_px"] = np.array(px)
    out["carm_scale_exact"] = np.array([R.pixel_scale(csc, cviews[3], 1, m, n) for m, n in px])
    out["carm_scale_cos"] = np.array([R.pixel_scale(csc, cviews[3], 0, m, n) for m, n in px])
    rng = np.random.default_rng(5)
    recs = []
    for t in range(12):
        i, j, k = (int(v) for v in rng.integers(0, 64, 3))
        v = int(rng.integers(0, 36))
        opts = (1, int(t % 2 == 0), 0, int(t % 3 != 0))
        rr, rc, rv, ri = R.collect_cut_records(csc, cviews[v], opts, i, j, k)
        for a, bb, c, d in zip(rr, rc, rv, ri):
            recs.append((t, i, j, k, v, *opts, a, bb, c, d))
    out["carm_records"] = np.array(recs, dtype=np.float64)
    # Siddon-K
    for K in (1, 2):
        out[f"SID_P_{K}"] = R.project_siddon(sc, x, K, threads=1)
        out[f"SID_BP_{K}"] = R.backproject_siddon(sc, b, K, threads=1)
    # solver
    out["adjoint_cvp_seed1"] = np.array(R.adjoint_test(sc, 0, (1, 1, 0, 1), 1, 1))
    out["adjoint_sid2_seed1"] = np.array(R.adjoint_test(sc, 1, (1, 1, 0, 1), 2, 1))
    xc, res = R.cgls(sc, b, 5)
    out["cgls_x"] = xc
    out["cgls_res"] = res
    out["rng_seed7_first16"] = R.fill_uniform01(16, 7)
    np.savez_compressed(os.path.join(HERE, "cvp_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "cvp_golden.npz"), sorted(out))


if __name__ == "__main__":
    main()
