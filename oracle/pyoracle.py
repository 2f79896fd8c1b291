"""ORACLE TEST INFRASTRUCTURE — not product code.

ctypes front-end for the two CPU checkers:

* ``Restatement`` — oracle/liboracle.so, the plain-C restatement of the
  reference hot path (oracle/cvp_oracle.c, each function citing the reference
  file:line it follows);
* ``Reference``   — oracle/_ref/libcbct_ref.so, the UNMODIFIED reference
  library (/root/reference/proj/src) compiled by oracle/Makefile behind our
  extern "C" shim (oracle/ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module. Both expose the same call signatures, so a test can run
the same case through either checker.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libcbct_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_ip) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class Scene:
    """Volume/detector/trajectory of one parity case (views as (V,17) doubles)."""
    counts: tuple
    voxel: tuple
    rows: int
    cols: int
    pw: float
    ph: float
    views: np.ndarray

    @property
    def n_views(self):
        return int(self.views.shape[0])

    def nvox(self):
        return int(np.prod(self.counts))

    def npx(self):
        return self.rows * self.cols * self.n_views


class _Checker:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        p = self.prefix
        self._last_error = getattr(self.lib, p + "last_error")
        self._last_error.restype = C.c_char_p

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._last_error().decode())

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def circular_trajectory(self, sid, sdd, n_views, arc_deg, rows, cols, pw, ph):
        out = np.zeros((n_views, 17))
        f = self._fn("make_circular_trajectory")
        f.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int,
                      C.c_double, C.c_double, _dp]
        self._check(f(sid, sdd, n_views, arc_deg, rows, cols, pw, ph, _d(out)))
        return out

    def fill_uniform01(self, n, seed):
        out = np.zeros(n)
        f = self._fn("fill_uniform01")
        f.argtypes = [_dp, C.c_size_t, C.c_uint64]
        rc = f(_d(out), n, seed)
        if isinstance(rc, int) and self.prefix == "ref_":
            self._check(rc)
        return out

    def pixel_scale(self, sc: Scene, view, exact, m, n):
        out = np.zeros(1)
        f = self._fn("pixel_scale")
        f.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, _dp]
        v = np.ascontiguousarray(view, dtype=np.float64)
        self._check(f(_d(v), sc.rows, sc.cols, sc.pw, sc.ph, int(exact), m, n, _d(out)))
        return float(out[0])

    def _geom(self, sc):
        return (np.asarray(sc.counts, dtype=np.int32), np.asarray(sc.voxel, dtype=np.float64),
                np.ascontiguousarray(sc.views, dtype=np.float64))

    def project_cvp(self, sc: Scene, vol, opts=(1, 1, 0, 1), threads=0):
        counts, voxel, views = self._geom(sc)
        vol = np.ascontiguousarray(vol, dtype=np.float64).ravel()
        out = np.zeros(sc.npx())
        o = np.asarray(opts, dtype=np.int32)
        if self.prefix == "ref_":
            f = self._fn("project_cvp")
            f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                          _ip, _ip, _dp, _dp, _dp]
            ex = np.asarray([threads, 0, 0], dtype=np.int32)
            self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                          _d(views), _i(o), _i(ex), _d(vol), _d(out), None))
        else:
            f = self._fn("project_cvp")
            f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                          _ip, _dp, _dp]
            self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                          _d(views), _i(o), _d(vol), _d(out)))
        return out.reshape(sc.n_views, sc.rows, sc.cols)

    def backproject_cvp(self, sc: Scene, proj, opts=(1, 1, 0, 1), threads=0):
        counts, voxel, views = self._geom(sc)
        proj = np.ascontiguousarray(proj, dtype=np.float64).ravel()
        out = np.zeros(sc.nvox())
        o = np.asarray(opts, dtype=np.int32)
        if self.prefix == "ref_":
            f = self._fn("backproject_cvp")
            f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                          _ip, _ip, _dp, _dp, _dp]
            ex = np.asarray([threads, 0, 0], dtype=np.int32)
            self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                          _d(views), _i(o), _i(ex), _d(proj), _d(out), None))
        else:
            f = self._fn("backproject_cvp")
            f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                          _ip, _dp, _dp]
            self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                          _d(views), _i(o), _d(proj), _d(out)))
        return out.reshape(sc.counts[2], sc.counts[1], sc.counts[0])

    def collect_cut_records(self, sc: Scene, view, opts, i, j, k, cap=256):
        counts, voxel, _ = self._geom(sc)
        v = np.ascontiguousarray(view, dtype=np.float64)
        rows = np.zeros(cap, dtype=np.int32)
        cols = np.zeros(cap, dtype=np.int32)
        vol = np.zeros(cap)
        inv = np.zeros(cap)
        n = np.zeros(1, dtype=np.int32)
        o = np.asarray(opts, dtype=np.int32)
        f = self._fn("collect_cut_records")
        f.argtypes = [_ip, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, _ip, C.c_int,
                      C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _dp, _ip]
        self._check(f(_i(counts), _d(voxel), _d(v), sc.rows, sc.cols, sc.pw, sc.ph, _i(o), i, j,
                      k, cap, _i(rows), _i(cols), _d(vol), _d(inv), _i(n)))
        c = min(int(n[0]), cap)
        return rows[:c], cols[:c], vol[:c], inv[:c]

    def project_siddon(self, sc: Scene, vol, k_per_edge, roi=None, threads=0):
        counts, voxel, views = self._geom(sc)
        vol = np.ascontiguousarray(vol, dtype=np.float64).ravel()
        out = np.zeros(sc.npx())
        r = np.asarray(roi, dtype=np.int32) if roi is not None else None
        if self.prefix == "ref_":
            f = self._fn("project_siddon")
            f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                          C.c_int, _ip, _ip, _dp, _dp]
            ex = np.asarray([threads, 0, 1], dtype=np.int32)
            self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                          _d(views), k_per_edge, _i(r), _i(ex), _d(vol), _d(out)))
        else:
            f = self._fn("project_siddon")
            f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                          C.c_int, _ip, _dp, _dp]
            self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                          _d(views), k_per_edge, _i(r), _d(vol), _d(out)))
        return out.reshape(sc.n_views, sc.rows, sc.cols)

    def backproject_siddon(self, sc: Scene, proj, k_per_edge, threads=0):
        counts, voxel, views = self._geom(sc)
        proj = np.ascontiguousarray(proj, dtype=np.float64).ravel()
        out = np.zeros(sc.nvox())
        if self.prefix == "ref_":
            f = self._fn("backproject_siddon")
            f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                          C.c_int, _ip, _dp, _dp]
            ex = np.asarray([threads, 0, 1], dtype=np.int32)
            self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                          _d(views), k_per_edge, _i(ex), _d(proj), _d(out)))
        else:
            f = self._fn("backproject_siddon")
            f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                          C.c_int, _dp, _dp]
            self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                          _d(views), k_per_edge, _d(proj), _d(out)))
        return out.reshape(sc.counts[2], sc.counts[1], sc.counts[0])


class Restatement(_Checker):
    prefix = "orc_"

    def __init__(self, path=RESTATEMENT_SO):
        super().__init__(path)

    # SF-TT (oracle/tt_oracle.c): Long, Fessler & Balter 2010, float64
    def project_tt(self, sc: Scene, vol, amplitude=1):
        counts, voxel, views = self._geom(sc)
        vol = np.ascontiguousarray(vol, dtype=np.float64).ravel()
        out = np.zeros(sc.npx())
        f = self._fn("project_tt")
        f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, _dp, _dp]
        self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.n_views, _d(views),
                      int(amplitude), _d(vol), _d(out)))
        return out.reshape(sc.n_views, sc.rows, sc.cols)

    def backproject_tt(self, sc: Scene, proj, amplitude=1):
        counts, voxel, views = self._geom(sc)
        proj = np.ascontiguousarray(proj, dtype=np.float64).ravel()
        out = np.zeros(sc.nvox())
        f = self._fn("backproject_tt")
        f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, _dp, _dp]
        self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.n_views, _d(views),
                      int(amplitude), _d(proj), _d(out)))
        return out.reshape(sc.counts[2], sc.counts[1], sc.counts[0])


class Reference(_Checker):
    prefix = "ref_"

    def __init__(self, path=REFERENCE_SO):
        super().__init__(path)

    def adjoint_test(self, sc: Scene, projector=0, opts=(1, 1, 0, 1), k_per_edge=1, seed=1):
        counts, voxel, views = self._geom(sc)
        out = np.zeros(1)
        o = np.asarray(opts, dtype=np.int32)
        f = self._fn("adjoint_test")
        f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp, C.c_int,
                      _ip, C.c_int, C.c_uint64, _dp]
        self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                      _d(views), projector, _i(o), k_per_edge, seed, _d(out)))
        return float(out[0])

    def cgls(self, sc: Scene, b, iterations, projector=0, opts=(1, 1, 0, 1), k_per_edge=1):
        counts, voxel, views = self._geom(sc)
        b = np.ascontiguousarray(b, dtype=np.float64).ravel()
        x = np.zeros(sc.nvox())
        res = np.zeros(iterations + 1)
        o = np.asarray(opts, dtype=np.int32)
        f = self._fn("cgls")
        f.argtypes = [_ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp, C.c_int,
                      _ip, C.c_int, _dp, C.c_int, _dp, _dp]
        self._check(f(_i(counts), _d(voxel), sc.rows, sc.cols, sc.pw, sc.ph, sc.n_views,
                      _d(views), projector, _i(o), k_per_edge, _d(b), iterations, _d(x), _d(res)))
        return x.reshape(sc.counts[2], sc.counts[1], sc.counts[0]), res


def restatement_available():
    return os.path.exists(RESTATEMENT_SO)


def reference_available():
    return os.path.exists(REFERENCE_SO)
