"""The cbctproj-compatible CLI (paper_2110_09841_b200/cli.py; reference
tools/commands.cpp). `compare` and argument handling run on CPU; the operator
subcommands run on the GPU (restating test_cli.cpp)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2110_09841_b200 as cb
from paper_2110_09841_b200 import cli, den

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    return subprocess.run([sys.executable, "-m", "paper_2110_09841_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_compare_reports_per_view_error(tmp_path):
    a = np.ones((3, 4, 5), np.float32)
    b = a.copy()
    b[1] *= 1.01
    den.den_write(tmp_path / "a.den", den.DenFile(4, 5, 3, a.ravel()))
    den.den_write(tmp_path / "b.den", den.DenFile(4, 5, 3, b.ravel()))
    rep = tmp_path / "r.csv"
    assert cli.main(["compare", str(tmp_path / "a.den"), str(tmp_path / "b.den"),
                     "--report", str(rep), "--arc", "360"]) == 0
    lines = open(rep).read().splitlines()
    assert lines[0] == "view,angle_deg,error_percent"
    assert abs(float(lines[2].split(",")[2]) - 1.0) < 1e-4
    assert lines[2].split(",")[1] == "120.000000"
    assert cli.main(["compare", str(tmp_path / "a.den"), str(tmp_path / "b.den"), "--tol", "0.5"]) == 1


def test_compare_dimension_mismatch(tmp_path):
    den.den_write(tmp_path / "a.den", den.DenFile(2, 2, 1, np.ones(4, np.float32)))
    den.den_write(tmp_path / "b.den", den.DenFile(2, 2, 2, np.ones(8, np.float32)))
    assert cli.main(["compare", str(tmp_path / "a.den"), str(tmp_path / "b.den")]) == 1


def test_parser_matches_reference_flags():
    ap = cli.build_parser()
    a = ap.parse_args(["project", "--volume", "v", "--output", "o", "--det-rows", "4", "--det-cols",
                       "4", "--circular", "541", "949", "36", "360", "--cos-scaling",
                       "--no-elevation-correction", "--relaxed"])
    o = cli._cvp_opts(a)
    assert o.scaling == cb.PixelScaling.Cos and not o.elevation_correction
    assert o.precision == cb.CvpPrecision.Single
    with pytest.raises(SystemExit):
        ap.parse_args(["project", "--volume", "v", "--output", "o", "--det-rows", "4",
                       "--det-cols", "4", "--cos-scaling", "--exact-scaling"])
    assert cli.view_angle_deg(3, 36, 360.0) == 30.0
    assert cli.view_angle_deg(99, 100, 198.0) == pytest.approx(198.0)


@pytest.mark.gpu
def test_project_backproject_recon_roundtrip(tmp_path):
    """test_cli.cpp:40-160: project a blob, backproject, reconstruct; CGLS
    residual falls and the DEN outputs have the right shapes."""
    geom = cb.VolumeGeometry.make((16, 16, 16), (1.0, 1.0, 1.0))
    k, j, i = np.meshgrid(*(np.arange(16),) * 3, indexing="ij")
    blob = np.exp(-((i - 7.5) ** 2 + (j - 7.5) ** 2 + (k - 7.5) ** 2) / 18.0)
    den.den_write(tmp_path / "vol.den", den.to_den(cb.AttenuationVolume(geom, blob.ravel())))
    traj = ["--circular", "40", "70", "24", "360"]
    r = _run(["project", "--volume", str(tmp_path / "vol.den"), "--output",
              str(tmp_path / "p.den"), "--det-rows", "32", "--det-cols", "32", *traj])
    assert r.returncode == 0, r.stderr
    p = den.den_read(tmp_path / "p.den")
    assert (p.dim_y, p.dim_x, p.dim_z) == (32, 32, 24)
    r = _run(["backproject", "--projections", str(tmp_path / "p.den"), "--output",
              str(tmp_path / "bp.den"), "--vol-dims", "16", "16", "16", *traj])
    assert r.returncode == 0, r.stderr
    r = _run(["recon", "--projections", str(tmp_path / "p.den"), "--output",
              str(tmp_path / "x.den"), "--vol-dims", "16", "16", "16", "--iterations", "20",
              "--residuals", str(tmp_path / "res.csv"), *traj])
    assert r.returncode == 0, r.stderr
    rows = open(tmp_path / "res.csv").read().splitlines()
    assert rows[0] == "iteration,residual_norm,relative_residual" and len(rows) == 22
    assert float(rows[-1].split(",")[2]) < 0.05


@pytest.mark.gpu
def test_bench_and_adjoint_test(tmp_path):
    csv = tmp_path / "b.csv"
    r = _run(["bench", "--preset", "desk", "--iterations", "1", "--csv", str(csv)])
    assert r.returncode == 0, r.stderr
    text = open(csv).read()
    assert "project_applications,,,1" in text and "backproject_applications,,,2" in text
    assert _run(["adjoint-test", "--preset", "desk", "--seeds", "2"]).returncode == 0
    assert _run(["adjoint-test", "--preset", "desk", "--projector", "siddon", "--siddon-k",
                 "2"]).returncode == 0
    # negative control: mismatched pair must fail
    assert _run(["adjoint-test", "--preset", "desk", "--mismatched-pair"]).returncode == 1
