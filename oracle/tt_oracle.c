/* ORACLE TEST INFRASTRUCTURE — not product code. See cvp_oracle.h for the
 * scene / view conventions.
 *
 * Separable-footprint projector with trapezoid/trapezoid footprints (SF-TT),
 * restated in float64 from the published algorithm: Y. Long, J. A. Fessler,
 * J. M. Balter, "3D forward and back-projection for X-ray CT using separable
 * footprints", IEEE Trans. Med. Imaging 29(11):1839-1850, 2010 — cited by the
 * reference paper (Tables I-II at :325,:347)
 * and left out of the reference implementation.
 * No third-party code exists here: the algorithm is restated from the paper's
 * formulas, for the flat-detector cone-beam geometry of the reference
 * (detector rows parallel to the x1x2 plane, geometry.cpp:52-88):
 *
 *   p(n, m) = sum_j mu_j * a_j(m) * F1_j(n) * F2_j(m)                 (SF model)
 *
 *   F1_j(n) = int_{n-1/2}^{n+1/2} trap(chi1; tau0..tau3) dchi1,   tau = chi1 of
 *             the 4 corners of voxel j's x1x2 footprint, sorted      (SF-TR/TT
 *             transaxial footprint, detector-cell averaged, in pixel units)
 *   F2_j(m) = int_{m-1/2}^{m+1/2} trap(chi2; t0..t3) dchi2,   t = chi2 of the
 *             voxel's z boundaries at its nearest and farthest corner depths,
 *             sorted                                              (SF-TT axial)
 *   a_j(m)  = l_phi0 * sqrt(1 + tan^2 theta)                    (amplitude)
 *             l_phi0 = min(a1 / |cos phi0|, a2 / |sin phi0|), phi0 the azimuth of
 *             the ray source -> voxel centre; tan theta = (chi2 - pp2) b2 /
 *             sqrt(u0^2 + f^2), u0 = (chi1(centre) - pp1) b1; A1: chi2 of the
 *             voxel centre, A2: chi2 = m (the detector row).
 *
 * chi1 and chi2 are evaluated directly from the pinhole model in world
 * coordinates (float64), independently of the device's voxel-local
 * formulation. The backprojector is the exact transpose. */
#include "cvp_oracle.h"

#include <math.h>
#include <stdlib.h>

typedef struct {
    double s[3], eu[3], ev[3], ew[3], f, pp1, pp2, b1, b2;
} tt_view;

static tt_view tt_unpack(const double* p) {
    tt_view v;
    for (int i = 0; i < 3; ++i) {
        v.s[i] = p[i];
        v.eu[i] = p[3 + i];
        v.ev[i] = p[6 + i];
        v.ew[i] = p[9 + i];
    }
    v.ev[0] = 0.0; /* e_v = (0, 0, -1) by construction (geometry.cpp:74-77) */
    v.ev[1] = 0.0;
    v.ev[2] = -1.0;
    v.f = p[12];
    v.pp1 = p[13];
    v.pp2 = p[14];
    v.b1 = p[15];
    v.b2 = p[16];
    return v;
}

/* pinhole projection of world point x: chi1, chi2 [px] and depth [mm] */
static void tt_project_point(const tt_view* v, const double x[3], double* chi1, double* chi2,
                             double* depth) {
    const double d[3] = {x[0] - v->s[0], x[1] - v->s[1], x[2] - v->s[2]};
    const double u = v->eu[0] * d[0] + v->eu[1] * d[1] + v->eu[2] * d[2];
    const double w = v->ev[0] * d[0] + v->ev[1] * d[1] + v->ev[2] * d[2];
    const double z = v->ew[0] * d[0] + v->ew[1] * d[1] + v->ew[2] * d[2];
    *depth = z;
    *chi1 = v->pp1 + v->f * u / (v->b1 * z);
    *chi2 = v->pp2 + v->f * w / (v->b2 * z);
}

static void tt_sort4(double t[4]) {
    for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b)
            if (t[b] < t[a]) {
                const double x = t[a];
                t[a] = t[b];
                t[b] = x;
            }
}

/* integral of the unit-height trapezoid (t0 <= t1 <= t2 <= t3) over (-inf, x] */
static double tt_trap_cdf(double x, const double t[4]) {
    double acc = 0.0;
    if (x > t[0]) { /* rising ramp */
        const double w = t[1] - t[0];
        const double c = x < t[1] ? x : t[1];
        if (w > 0.0) acc += 0.5 * (c - t[0]) * (c - t[0]) / w;
    }
    if (x > t[1]) acc += (x < t[2] ? x : t[2]) - t[1]; /* plateau */
    if (x > t[2]) { /* falling ramp */
        const double w = t[3] - t[2];
        const double c = x < t[3] ? x : t[3];
        if (w > 0.0) acc += (c - t[2]) * (w - 0.5 * (c - t[2])) / w;
    }
    return acc;
}

/* cell average of the trapezoid over [k - 1/2, k + 1/2] (pixel units) */
static double tt_cell(int k, const double t[4]) {
    return tt_trap_cdf(k + 0.5, t) - tt_trap_cdf(k - 0.5, t);
}

typedef void (*tt_sink)(void* ctx, size_t vox, size_t px, double w);

static int tt_walk(const int* counts, const double* voxel, int rows, int cols, int n_views,
                   const double* views17, int amplitude, tt_sink sink, void* ctx) {
    const int N1 = counts[0], N2 = counts[1], N3 = counts[2];
    const double a1 = voxel[0], a2 = voxel[1], a3 = voxel[2];
    const double mn[3] = {-0.5 * N1 * a1, -0.5 * N2 * a2, -0.5 * N3 * a3};
    double* f1 = malloc(sizeof(double) * (size_t)cols);
    double* f2 = malloc(sizeof(double) * (size_t)rows);
    if (!f1 || !f2) {
        free(f1);
        free(f2);
        return 2;
    }
    for (int vi = 0; vi < n_views; ++vi) {
        const tt_view v = tt_unpack(views17 + 17 * vi);
        const size_t vbase = (size_t)vi * rows * cols;
        for (int j = 0; j < N2; ++j)
            for (int i = 0; i < N1; ++i) {
                const double xc = mn[0] + (i + 0.5) * a1, yc = mn[1] + (j + 0.5) * a2;
                /* transaxial trapezoid: chi1 of the 4 footprint corners (any z) */
                double tau[4], dep[4];
                for (int q = 0; q < 4; ++q) {
                    const double x[3] = {xc + ((q & 1) ? 0.5 : -0.5) * a1,
                                         yc + ((q & 2) ? 0.5 : -0.5) * a2, 0.0};
                    double c2;
                    tt_project_point(&v, x, &tau[q], &c2, &dep[q]);
                    if (!(dep[q] > 0.0)) {
                        free(f1);
                        free(f2);
                        return 2; /* voxel base behind the source plane */
                    }
                }
                tt_sort4(tau);
                double dn = dep[0], df = dep[0];
                for (int q = 1; q < 4; ++q) {
                    dn = dep[q] < dn ? dep[q] : dn;
                    df = dep[q] > df ? dep[q] : df;
                }
                int nlo = (int)ceil(tau[0] - 0.5), nhi = (int)floor(tau[3] + 0.5);
                if (nlo < 0) nlo = 0;
                if (nhi > cols - 1) nhi = cols - 1;
                if (nlo > nhi) continue;
                for (int n = nlo; n <= nhi; ++n) f1[n] = tt_cell(n, tau);
                /* amplitude: l_phi0 of the central ray, elevation term */
                double cchi1, cchi2_unused, cdep;
                const double xcen[3] = {xc, yc, 0.0};
                tt_project_point(&v, xcen, &cchi1, &cchi2_unused, &cdep);
                const double rx = xc - v.s[0], ry = yc - v.s[1];
                const double rho = sqrt(rx * rx + ry * ry);
                const double cphi = fabs(rx) / rho, sphi = fabs(ry) / rho;
                const double l1 = cphi > 0.0 ? a1 / cphi : INFINITY;
                const double l2 = sphi > 0.0 ? a2 / sphi : INFINITY;
                const double lphi = l1 < l2 ? l1 : l2;
                const double u0 = (cchi1 - v.pp1) * v.b1;
                const double den = u0 * u0 + v.f * v.f;
                for (int k = 0; k < N3; ++k) {
                    const double zc = mn[2] + (k + 0.5) * a3;
                    /* axial trapezoid: chi2 of z_lo / z_hi at the near / far depths */
                    double t[4];
                    const double zs[2] = {zc - 0.5 * a3, zc + 0.5 * a3}, ds[2] = {dn, df};
                    for (int q = 0; q < 4; ++q)
                        t[q] = v.pp2 - (zs[q & 1] - v.s[2]) * v.f / (v.b2 * ds[q >> 1]);
                    tt_sort4(t);
                    int mlo = (int)ceil(t[0] - 0.5), mhi = (int)floor(t[3] + 0.5);
                    if (mlo < 0) mlo = 0;
                    if (mhi > rows - 1) mhi = rows - 1;
                    if (mlo > mhi) continue;
                    const size_t vox = ((size_t)k * N2 + j) * N1 + i;
                    /* A1: elevation of the voxel centre's projection */
                    double cc1, cc2, cd;
                    const double xv[3] = {xc, yc, zc};
                    tt_project_point(&v, xv, &cc1, &cc2, &cd);
                    const double tv = (cc2 - v.pp2) * v.b2;
                    const double amp_a1 = lphi * sqrt(1.0 + tv * tv / den);
                    for (int m = mlo; m <= mhi; ++m) {
                        f2[m] = tt_cell(m, t);
                        if (!(f2[m] > 0.0)) continue;
                        const double tm = (m - v.pp2) * v.b2;
                        const double amp = amplitude ? lphi * sqrt(1.0 + tm * tm / den) : amp_a1;
                        for (int n = nlo; n <= nhi; ++n)
                            if (f1[n] > 0.0)
                                sink(ctx, vox, vbase + (size_t)m * cols + n, amp * f1[n] * f2[m]);
                    }
                }
            }
    }
    free(f1);
    free(f2);
    return 0;
}

typedef struct {
    const double* in;
    double* out;
} tt_io;

static void tt_fwd_sink(void* c, size_t vox, size_t px, double w) {
    tt_io* io = (tt_io*)c;
    io->out[px] += io->in[vox] * w;
}

static void tt_bwd_sink(void* c, size_t vox, size_t px, double w) {
    tt_io* io = (tt_io*)c;
    io->out[vox] += io->in[px] * w;
}

int orc_project_tt(const int* counts, const double* voxel, int rows, int cols, int n_views,
                   const double* views17, int amplitude, const double* vol, double* out) {
    const size_t np = (size_t)rows * cols * n_views;
    for (size_t q = 0; q < np; ++q) out[q] = 0.0;
    tt_io io = {vol, out};
    return tt_walk(counts, voxel, rows, cols, n_views, views17, amplitude, tt_fwd_sink, &io);
}

int orc_backproject_tt(const int* counts, const double* voxel, int rows, int cols, int n_views,
                       const double* views17, int amplitude, const double* proj, double* out) {
    const size_t nv = (size_t)counts[0] * counts[1] * counts[2];
    for (size_t q = 0; q < nv; ++q) out[q] = 0.0;
    tt_io io = {proj, out};
    return tt_walk(counts, voxel, rows, cols, n_views, views17, amplitude, tt_bwd_sink, &io);
}
