"""Shared fixtures. GPU tests are marked ``gpu``; everything else runs on CPU.

Checkers (test infrastructure only): oracle/_ref/libcbct_ref.so — the
reference compiled from its sources — and oracle/liboracle.so — the plain-C
restatement, pinned against the reference and tests/golden/.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def checker():
    """The strongest CPU checker available: the compiled reference if present,
    else the C restatement."""
    from oracle import pyoracle
    if pyoracle.reference_available():
        return pyoracle.Reference()
    return pyoracle.Restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle import pyoracle
    if not pyoracle.reference_available():
        pytest.skip("oracle/_ref not built")
    return pyoracle.Reference()


@pytest.fixture(scope="session")
def restatement():
    from oracle import pyoracle
    return pyoracle.Restatement()


def rel_l2(got, ref):
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    return float(np.linalg.norm(got - ref) / np.linalg.norm(ref))


def max_rel(got, ref):
    """max|delta| / max|ref| (the well-conditioned 'max relative error')."""
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    return float(np.abs(got - ref).max() / np.abs(ref).max())


def make_case(counts, voxel, rows, cols, pw, ph, sid, sdd, n_views, arc=360.0, device=0):
    """(DeviceScene | None, oracle Scene, views) for one parity case."""
    import paper_2110_09841_b200 as cb
    from oracle.pyoracle import Scene
    det = cb.DetectorGeometry.make(rows, cols, pw, ph)
    geom = cb.VolumeGeometry.make(counts, voxel)
    views = cb.make_circular_trajectory(sid, sdd, n_views, arc, det)
    sc = Scene(tuple(counts), tuple(voxel), rows, cols, pw, ph, cb.views_to_array(views))
    return geom, det, views, sc
