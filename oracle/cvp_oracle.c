/* ORACLE TEST INFRASTRUCTURE — not product code. See cvp_oracle.h.
 *
 * Plain-C restatement of the reference (/root/reference/proj) hot path.
 * Serial, scalar; used by tests/ as an independent checker and by bench.py as
 * the "port" CPU baseline when oracle/_ref is unavailable. */
#include "cvp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
static void orc_set_error(const char* msg) { snprintf(g_err, sizeof g_err, "%s", msg); }
const char* orc_last_error(void) { return g_err; }

/* ---------------- mt19937_64 + uniform01 (solver.hpp:27, solver.cpp:30-33) ---- */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (s->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
        s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        s->mti = 0;
    }
    uint64_t x = s->mt[s->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

void orc_fill_uniform01(double* out, size_t n, uint64_t seed) {
    mt64 s;
    mt64_seed(&s, seed);
    for (size_t i = 0; i < n; ++i) out[i] = (double)(mt64_next(&s) >> 11) * 0x1.0p-53;
}

/* ---------------- views (geometry.hpp:70-123, geometry.cpp:52-88) ---------- */
typedef struct {
    double s[3], eu[3], ev[3], ew[3], f, pp1, pp2, b1, b2;
} orc_view;

static orc_view view_unpack(const double* p) {
    orc_view v;
    for (int i = 0; i < 3; ++i) {
        v.s[i] = p[i];
        v.eu[i] = p[3 + i];
        v.ev[i] = p[6 + i];
        v.ew[i] = p[9 + i];
    }
    /* ViewGeometry::make snaps e_v onto (0,0,-1) (geometry.cpp:74-77) */
    v.ev[0] = 0.0;
    v.ev[1] = 0.0;
    v.ev[2] = -1.0;
    v.f = p[12];
    v.pp1 = p[13];
    v.pp2 = p[14];
    v.b1 = p[15];
    v.b2 = p[16];
    return v;
}

/* make_circular_trajectory (geometry.cpp:182-210). */
int orc_make_circular_trajectory(double sid, double sdd, int n_views, double arc_deg, int rows,
                                 int cols, double pw, double ph, double* out17) {
    if (n_views <= 0) {
        orc_set_error("need at least one view");
        return 1;
    }
    if (!(sid > 0.0) || !(sdd > 0.0)) {
        orc_set_error("distances must be positive");
        return 1;
    }
    if (!(arc_deg > 0.0) || arc_deg > 360.0) {
        orc_set_error("arc must lie in (0, 360] degrees");
        return 1;
    }
    double step = fabs(arc_deg - 360.0) < 1e-9 ? 360.0 / n_views
                                                : (n_views > 1 ? arc_deg / (n_views - 1) : 0.0);
    for (int v = 0; v < n_views; ++v) {
        double w = v * step * M_PI / 180.0;
        double c = cos(w), s = sin(w);
        double* p = out17 + 17 * v;
        p[0] = sid * c;
        p[1] = sid * s;
        p[2] = 0.0;
        /* e_w = (-c,-s,0), e_v = (0,0,-1), e_u = e_v x e_w */
        double ew[3] = {-c, -s, 0.0}, ev[3] = {0.0, 0.0, -1.0};
        p[3] = ev[1] * ew[2] - ev[2] * ew[1];
        p[4] = ev[2] * ew[0] - ev[0] * ew[2];
        p[5] = ev[0] * ew[1] - ev[1] * ew[0];
        p[6] = ev[0];
        p[7] = ev[1];
        p[8] = ev[2];
        p[9] = ew[0];
        p[10] = ew[1];
        p[11] = ew[2];
        p[12] = sdd;
        p[13] = (cols - 1) * 0.5;
        p[14] = (rows - 1) * 0.5;
        p[15] = pw;
        p[16] = ph;
    }
    return 0;
}

/* ---------------- pixel scaling (cvp.cpp:251-302, 570-605) ---------------- */
static int spherical_quad(const double t[4][3], double* out) {
    double nrm[4][3];
    for (int i = 0; i < 4; ++i) {
        double l = sqrt(t[i][0] * t[i][0] + t[i][1] * t[i][1] + t[i][2] * t[i][2]);
        if (fabs(l - 1.0) > 1e-12) {
            orc_set_error("spherical quad vertices must be unit vectors");
            return 1;
        }
    }
    for (int i = 0; i < 4; ++i) {
        const double* a = t[i];
        const double* b = t[(i + 1) % 4];
        nrm[i][0] = a[1] * b[2] - a[2] * b[1];
        nrm[i][1] = a[2] * b[0] - a[0] * b[2];
        nrm[i][2] = a[0] * b[1] - a[1] * b[0];
        double q = nrm[i][0] * nrm[i][0] + nrm[i][1] * nrm[i][1] + nrm[i][2] * nrm[i][2];
        if (q < 1e-30) {
            orc_set_error("degenerate spherical quad (parallel consecutive vertices)");
            return 4;
        }
        double l = sqrt(q);
        for (int d = 0; d < 3; ++d) nrm[i][d] /= l;
    }
    double sum = 0.0;
    for (int i = 0; i < 4; ++i) {
        const double* a = nrm[i];
        const double* b = nrm[(i + 1) % 4];
        double c = a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
        if (c < -1.0) c = -1.0;
        if (c > 1.0) c = 1.0;
        sum += acos(c);
    }
    double area = 2.0 * M_PI - sum;
    if (!(area > 0.0) || !(area < 4.0 * M_PI)) {
        orc_set_error("spherical quad area outside (0, 4*pi)");
        return 4;
    }
    *out = area;
    return 0;
}

static void unit3(double x, double y, double z, double* o) {
    double l = sqrt(x * x + y * y + z * z);
    o[0] = x / l;
    o[1] = y / l;
    o[2] = z / l;
}

static int scale_at(const orc_view* v, int exact, int m, int n, double* out) {
    if (!exact) {
        double u = (n - v->pp1) * v->b1, w = (m - v->pp2) * v->b2;
        double c = v->f / sqrt(u * u + w * w + v->f * v->f);
        *out = v->f * v->f / (v->b1 * v->b2 * c * c * c);
        return 0;
    }
    double u0 = (n - 0.5 - v->pp1) * v->b1, u1 = (n + 0.5 - v->pp1) * v->b1;
    double w0 = (m - 0.5 - v->pp2) * v->b2, w1 = (m + 0.5 - v->pp2) * v->b2;
    double t[4][3];
    unit3(u0, w0, v->f, t[0]);
    unit3(u1, w0, v->f, t[1]);
    unit3(u1, w1, v->f, t[2]);
    unit3(u0, w1, v->f, t[3]);
    double omega;
    int rc = spherical_quad(t, &omega);
    if (rc) return rc;
    *out = 1.0 / omega;
    return 0;
}

static int orc_scale_image(const orc_view* v, int rows, int cols, int exact, double* img) {
    for (int m = 0; m < rows; ++m)
        for (int n = 0; n < cols; ++n) {
            int rc = scale_at(v, exact, m, n, &img[(size_t)m * cols + n]);
            if (rc) return rc;
        }
    return 0;
}

int orc_pixel_scale(const double* view17, int rows, int cols, double pw, double ph, int exact,
                    int m, int n, double* out) {
    (void)pw;
    (void)ph;
    if (m < 0 || n < 0 || m >= rows || n >= cols) {
        orc_set_error("pixel outside the detector");
        return 3;
    }
    orc_view v = view_unpack(view17);
    return scale_at(&v, exact, m, n, out);
}

/* ---------------- CVP body, instantiated for double and float ------------- */
#define R double
#define FN(x) x##_d
#define RABS fabs
#define RSQRT sqrt
#include "cvp_oracle_body.inc"
#undef R
#undef FN
#undef RABS
#undef RSQRT

#define R float
#define FN(x) x##_f
#define RABS fabsf
#define RSQRT sqrtf
#include "cvp_oracle_body.inc"
#undef R
#undef FN
#undef RABS
#undef RSQRT

/* check_view_consistency (cvp.cpp:237-247). */
static int check_views(const int* counts, const double* a, double pw, double ph, int n_views,
                       const orc_view* views) {
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = counts[d] * a[d] * -0.5;
        hi[d] = lo[d] + counts[d] * a[d];
    }
    for (int v = 0; v < n_views; ++v) {
        if (fabs(views[v].b1 - pw) > 1e-9 || fabs(views[v].b2 - ph) > 1e-9) {
            orc_set_error("view pixel size does not match the detector geometry");
            return 1;
        }
        const double* s = views[v].s;
        if (s[0] > lo[0] && s[0] < hi[0] && s[1] > lo[1] && s[1] < hi[1] && s[2] > lo[2] &&
            s[2] < hi[2]) {
            orc_set_error("unsupported configuration: source inside the volume box");
            return 2;
        }
    }
    return 0;
}

static orc_view* unpack_all(const double* views17, int n) {
    orc_view* v = (orc_view*)malloc(sizeof(orc_view) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) v[i] = view_unpack(views17 + 17 * i);
    return v;
}

int orc_project_cvp(const int* counts, const double* voxel, int rows, int cols, double pw,
                    double ph, int n_views, const double* views17, const int* opts4,
                    const double* vol, double* out) {
    orc_view* views = unpack_all(views17, n_views);
    int rc = check_views(counts, voxel, pw, ph, n_views, views);
    if (!rc)
        rc = opts4[2] ? project_f(counts, voxel, rows, cols, n_views, views, opts4, vol, out)
                      : project_d(counts, voxel, rows, cols, n_views, views, opts4, vol, out);
    free(views);
    return rc;
}

int orc_backproject_cvp(const int* counts, const double* voxel, int rows, int cols, double pw,
                        double ph, int n_views, const double* views17, const int* opts4,
                        const double* proj, double* out) {
    orc_view* views = unpack_all(views17, n_views);
    int rc = check_views(counts, voxel, pw, ph, n_views, views);
    if (!rc)
        rc = opts4[2] ? backproject_f(counts, voxel, rows, cols, n_views, views, opts4, proj, out)
                      : backproject_d(counts, voxel, rows, cols, n_views, views, opts4, proj, out);
    free(views);
    return rc;
}

/* collect_cut_records (cvp.cpp:652-689): double precision, no detector clamping. */
typedef struct {
    int cap, count;
    int *rows, *cols;
    double *vol, *invr2;
} rec_user;

static void rec_sink(void* u, int m, int n, double volume, double inv_r2) {
    rec_user* r = (rec_user*)u;
    if (r->count < r->cap) {
        r->rows[r->count] = m;
        r->cols[r->count] = n;
        r->vol[r->count] = volume;
        r->invr2[r->count] = inv_r2;
    }
    r->count++;
}

int orc_collect_cut_records(const int* counts, const double* voxel, const double* view17,
                            int rows, int cols, double pw, double ph, const int* opts4, int i,
                            int j, int k, int cap, int* rows_out, int* cols_out,
                            double* vol_out, double* invr2_out, int* n_out) {
    if (i < 0 || j < 0 || k < 0 || i >= counts[0] || j >= counts[1] || k >= counts[2]) {
        orc_set_error("voxel index outside lattice");
        return 3;
    }
    orc_view v = view_unpack(view17);
    int rc = check_views(counts, voxel, pw, ph, 1, &v);
    if (rc) return rc;
    ctx_t_d c = ctx_make_d(&v, rows, cols);
    double bcx, bcy;
    poly_d base = base_square_d(counts, voxel, i, j, &bcx, &bcy);
    cut_d cuts[ORC_MAX_CUTS];
    int nc = compute_cuts_d(&c, &base, 0, opts4[1] != 0, cuts, ORC_MAX_CUTS);
    if (nc == -2) {
        orc_set_error("numerical degeneracy: voxel base reaches the source plane");
        return 2;
    }
    if (nc < 0 || nc > ORC_MAX_CUTS) {
        orc_set_error("degenerate cut");
        return 4;
    }
    double minz = counts[2] * voxel[2] * -0.5;
    double zc = minz + (k + 0.5) * voxel[2];
    double z_lo = zc - 0.5 * voxel[2], z_hi = zc + 0.5 * voxel[2];
    double dz = zc - c.s3;
    double inv_r2_fixed = -1.0;
    if (opts4[3] == 0) {
        double rx = bcx - c.sx, ry = bcy - c.sy;
        inv_r2_fixed = 1.0 / (rx * rx + ry * ry + dz * dz);
    }
    rec_user u = {cap, 0, rows_out, cols_out, vol_out, invr2_out};
    for (int q = 0; q < nc; ++q) {
        int on = opts4[1] && cuts[q].halfw > 0.0 && dz * dz > cuts[q].rho2 * 1e-28;
        visit_rows_d(&c, &cuts[q], z_lo, z_hi, on, 0, inv_r2_fixed, rec_sink, &u);
    }
    *n_out = u.count;
    return 0;
}

/* ---------------- Siddon-K (siddon.cpp:21-313) ---------------------------- */
typedef struct {
    double lo[3], a[3];
    int i0[3], n[3];
} orc_box;

typedef void (*ray_sink)(void* user, int i, int j, int k, double chord);

/* traverse (siddon.cpp:37-98). */
static void traverse(const orc_box* b, const double* s, const double* d, double dlen,
                     ray_sink emit, void* user) {
    double t0 = 0.0, t1 = INFINITY;
    for (int ax = 0; ax < 3; ++ax) {
        double hi = b->lo[ax] + b->a[ax] * b->n[ax];
        if (d[ax] == 0.0) {
            if (s[ax] < b->lo[ax] || s[ax] >= hi) return;
        } else {
            double ta = (b->lo[ax] - s[ax]) / d[ax];
            double tb = (hi - s[ax]) / d[ax];
            if (ta > tb) {
                double x = ta;
                ta = tb;
                tb = x;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
    }
    if (!(t0 < t1)) return;
    int idx[3], step[3];
    double tnext[3], tdelta[3];
    for (int ax = 0; ax < 3; ++ax) {
        double pos = s[ax] + t0 * d[ax];
        int q = (int)floor((pos - b->lo[ax]) / b->a[ax]);
        if (q < 0) q = 0;
        if (q > b->n[ax] - 1) q = b->n[ax] - 1;
        idx[ax] = q;
        if (d[ax] > 0.0) {
            step[ax] = 1;
            tnext[ax] = (b->lo[ax] + (idx[ax] + 1) * b->a[ax] - s[ax]) / d[ax];
            tdelta[ax] = b->a[ax] / d[ax];
        } else if (d[ax] < 0.0) {
            step[ax] = -1;
            tnext[ax] = (b->lo[ax] + idx[ax] * b->a[ax] - s[ax]) / d[ax];
            tdelta[ax] = -b->a[ax] / d[ax];
        } else {
            step[ax] = 0;
            tnext[ax] = INFINITY;
            tdelta[ax] = INFINITY;
        }
    }
    double t = t0;
    for (;;) {
        double tn = tnext[0];
        if (tnext[1] < tn) tn = tnext[1];
        if (tnext[2] < tn) tn = tnext[2];
        double len = ((tn < t1 ? tn : t1) - t) * dlen;
        if (len > 0.0) emit(user, b->i0[0] + idx[0], b->i0[1] + idx[1], b->i0[2] + idx[2], len);
        if (tn >= t1) return;
        int left = 0;
        for (int ax = 0; ax < 3; ++ax) {
            if (tnext[ax] == tn) {
                idx[ax] += step[ax];
                if (idx[ax] < 0 || idx[ax] >= b->n[ax]) left = 1;
                tnext[ax] += tdelta[ax];
            }
        }
        if (left) return;
        t = tn;
    }
}

typedef struct {
    const double* mu;
    double* dst;
    size_t n1, n2;
    double acc, w;
} sid_user;

static void sid_fwd(void* u, int i, int j, int k, double chord) {
    sid_user* s = (sid_user*)u;
    s->acc += s->mu[((size_t)k * s->n2 + j) * s->n1 + i] * chord;
}
static void sid_bwd(void* u, int i, int j, int k, double chord) {
    sid_user* s = (sid_user*)u;
    s->dst[((size_t)k * s->n2 + j) * s->n1 + i] += s->w * chord;
}

/* DetectorPlane (siddon.cpp:135-150). */
static void det_plane(const orc_view* v, double* base, double* du, double* dv) {
    for (int d = 0; d < 3; ++d) {
        du[d] = v->b1 * v->eu[d];
        dv[d] = v->b2 * v->ev[d];
    }
    for (int d = 0; d < 3; ++d) base[d] = v->s[d] + v->f * v->ew[d] - v->pp1 * du[d] - v->pp2 * dv[d];
}

static int check_siddon(const int* counts, const double* a, double pw, double ph, int n_views,
                        const orc_view* views, int K) {
    if (K < 1) {
        orc_set_error("Siddon K must be at least 1");
        return 1;
    }
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = counts[d] * a[d] * -0.5;
        hi[d] = lo[d] + counts[d] * a[d];
    }
    for (int v = 0; v < n_views; ++v) {
        if (fabs(views[v].b1 - pw) > 1e-9 || fabs(views[v].b2 - ph) > 1e-9) {
            orc_set_error("view pixel size does not match the detector geometry");
            return 1;
        }
        const double* s = views[v].s;
        if (s[0] > lo[0] && s[0] < hi[0] && s[1] > lo[1] && s[1] < hi[1] && s[2] > lo[2] &&
            s[2] < hi[2]) {
            orc_set_error("unsupported configuration: source inside the volume box");
            return 2;
        }
    }
    return 0;
}

static int clampi(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

int orc_project_siddon(const int* counts, const double* voxel, int rows, int cols, double pw,
                       double ph, int n_views, const double* views17, int K, const int* roi4,
                       const double* vol, double* out) {
    orc_view* views = unpack_all(views17, n_views);
    int rc = check_siddon(counts, voxel, pw, ph, n_views, views, K);
    if (rc) {
        free(views);
        return rc;
    }
    size_t npx = (size_t)rows * cols;
    memset(out, 0, npx * (size_t)n_views * sizeof(double));
    /* tight nonzero sub-box (siddon.cpp:182-211) */
    int blo[3] = {counts[0], counts[1], counts[2]}, bhi[3] = {0, 0, 0};
    const size_t n1 = counts[0], n2 = counts[1];
    for (int k = 0; k < counts[2]; ++k)
        for (int j = 0; j < counts[1]; ++j)
            for (int i = 0; i < counts[0]; ++i)
                if (vol[((size_t)k * n2 + j) * n1 + i] != 0.0) {
                    int q[3] = {i, j, k};
                    for (int d = 0; d < 3; ++d) {
                        if (q[d] < blo[d]) blo[d] = q[d];
                        if (q[d] + 1 > bhi[d]) bhi[d] = q[d] + 1;
                    }
                }
    if (bhi[0] <= blo[0]) {
        free(views);
        return 0;
    }
    orc_box box;
    for (int d = 0; d < 3; ++d) {
        box.a[d] = voxel[d];
        box.i0[d] = blo[d];
        box.n[d] = bhi[d] - blo[d];
        box.lo[d] = counts[d] * voxel[d] * -0.5 + blo[d] * voxel[d];
    }
    int r0 = 0, r1 = rows, c0 = 0, c1 = cols;
    if (roi4) {
        r0 = clampi(roi4[0], 0, rows);
        r1 = roi4[1] < 0 ? rows : clampi(roi4[1], r0, rows);
        c0 = clampi(roi4[2], 0, cols);
        c1 = roi4[3] < 0 ? cols : clampi(roi4[3], c0, cols);
    }
    double inv_k2 = 1.0 / ((double)K * (double)K);
    for (int v = 0; v < n_views; ++v) {
        double base[3], du[3], dv[3];
        det_plane(&views[v], base, du, dv);
        const double* src = views[v].s;
        double* img = out + (size_t)v * npx;
        for (int m = r0; m < r1; ++m)
            for (int n = c0; n < c1; ++n) {
                sid_user u = {vol, NULL, n1, n2, 0.0, 0.0};
                for (int uu = 0; uu < K; ++uu) {
                    double chi1 = n + (uu + 0.5) / K - 0.5;
                    for (int ww = 0; ww < K; ++ww) {
                        double chi2 = m + (ww + 0.5) / K - 0.5;
                        double dir[3];
                        for (int d = 0; d < 3; ++d)
                            dir[d] = base[d] + chi1 * du[d] + chi2 * dv[d] - src[d];
                        double dl = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
                        traverse(&box, src, dir, dl, sid_fwd, &u);
                    }
                }
                img[(size_t)m * cols + n] = u.acc * inv_k2;
            }
    }
    free(views);
    return 0;
}

int orc_backproject_siddon(const int* counts, const double* voxel, int rows, int cols, double pw,
                           double ph, int n_views, const double* views17, int K,
                           const double* proj, double* out) {
    orc_view* views = unpack_all(views17, n_views);
    int rc = check_siddon(counts, voxel, pw, ph, n_views, views, K);
    if (rc) {
        free(views);
        return rc;
    }
    const size_t n1 = counts[0], n2 = counts[1];
    memset(out, 0, n1 * n2 * (size_t)counts[2] * sizeof(double));
    orc_box box;
    for (int d = 0; d < 3; ++d) {
        box.a[d] = voxel[d];
        box.i0[d] = 0;
        box.n[d] = counts[d];
        box.lo[d] = counts[d] * voxel[d] * -0.5;
    }
    size_t npx = (size_t)rows * cols;
    double inv_k2 = 1.0 / ((double)K * (double)K);
    for (int v = 0; v < n_views; ++v) {
        double base[3], du[3], dv[3];
        det_plane(&views[v], base, du, dv);
        const double* src = views[v].s;
        const double* img = proj + (size_t)v * npx;
        for (int m = 0; m < rows; ++m)
            for (int n = 0; n < cols; ++n) {
                double w = img[(size_t)m * cols + n] * inv_k2;
                if (w == 0.0) continue;
                sid_user u = {NULL, out, n1, n2, 0.0, w};
                for (int uu = 0; uu < K; ++uu) {
                    double chi1 = n + (uu + 0.5) / K - 0.5;
                    for (int ww = 0; ww < K; ++ww) {
                        double chi2 = m + (ww + 0.5) / K - 0.5;
                        double dir[3];
                        for (int d = 0; d < 3; ++d)
                            dir[d] = base[d] + chi1 * du[d] + chi2 * dv[d] - src[d];
                        double dl = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
                        traverse(&box, src, dir, dl, sid_bwd, &u);
                    }
                }
            }
    }
    free(views);
    return 0;
}

double orc_dot_kahan(const double* a, const double* b, size_t n) {
    double sum = 0.0, c = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double y = a[i] * b[i] - c;
        double t = sum + y;
        c = (t - sum) - y;
        sum = t;
    }
    return sum;
}
