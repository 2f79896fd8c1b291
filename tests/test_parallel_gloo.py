"""World-size-2 gloo test of the multi-GPU partitioning: view
shards + reduce-scatter over z-slabs + distributed CGLS equal the
single-process results."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def gloo_results(tmp_path_factory):
    out = tmp_path_factory.mktemp("gloo")
    port = _free_port()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_gloo_worker.py"), str(r), "2",
                               str(port), str(out)]) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    return [dict(np.load(out / f"rank{r}.npz")) for r in range(2)]


def _single(restatement):
    from oracle.pyoracle import Scene
    views = restatement.circular_trajectory(40.0, 70.0, 8, 360.0, 32, 32, 1.0, 1.0)
    sc = Scene((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, views)
    x = restatement.fill_uniform01(16 ** 3, 7).astype(np.float32).astype(np.float64)
    b = restatement.fill_uniform01(32 * 32 * 8, 8).astype(np.float32).astype(np.float64)
    return sc, restatement.project_cvp(sc, x), restatement.backproject_cvp(sc, b).ravel()


def test_forward_shards_are_the_full_projection(gloo_results, restatement):
    _, p_full, _ = _single(restatement)
    got = np.concatenate([r["p_local"] for r in gloo_results])
    assert [int(r["vc"]) for r in gloo_results] == [4, 4]
    assert np.abs(got - p_full).max() <= 1e-5 * np.abs(p_full).max()


def test_reduce_scatter_slabs_sum_the_partials(gloo_results, restatement):
    _, _, bp = _single(restatement)
    for r in gloo_results:
        b0, b1 = (int(t) for t in r["slab_range"])
        assert np.abs(r["slab"][: b1 - b0] - bp[b0:b1]).max() <= 1e-5 * np.abs(bp).max()
        assert np.abs(r["full"] - bp).max() <= 1e-5 * np.abs(bp).max()
    # slabs are contiguous z ranges: rank 0 holds k < 8, rank 1 k >= 8
    assert [tuple(int(t) for t in r["slab_range"]) for r in gloo_results] == [(0, 2048), (2048, 4096)]


def test_distributed_cgls_matches_single_process(gloo_results, checker):
    from oracle.pyoracle import Scene
    views = checker.circular_trajectory(40.0, 70.0, 8, 360.0, 32, 32, 1.0, 1.0)
    sc = Scene((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, views)
    b = checker.fill_uniform01(32 * 32 * 8, 8).astype(np.float32).astype(np.float64)
    if hasattr(checker, "cgls"):
        x_ref, res_ref = checker.cgls(sc, b, 4)
    else:
        pytest.skip("single-process CGLS needs the compiled reference")
    for r in gloo_results:
        np.testing.assert_allclose(r["cgls_res"], res_ref, rtol=1e-4)
        assert np.linalg.norm(r["cgls_x"] - x_ref.ravel()) <= 1e-3 * np.linalg.norm(x_ref)
