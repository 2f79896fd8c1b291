// Device-side CVP geometry: column cuts (float64 in exact mode, float32 in
// relaxed mode) and the per-voxel row walk in voxel-local float32 coordinates.
//
// Reference algorithm: /root/reference/proj/src/cvp.cpp (ViewCtx :26-70,
// BandCutter :73-98, fill_cut_info :111-136, compute_cuts :138-157,
// clamp_mean :161-175, visit_rows :180-235, process_column :326-349) and the
// polygon kernel in include/cbct/polygon.hpp:101-164.
//
// B200 re-design:
//  * The cut geometry of one voxel column under one view is computed ONCE per
//    CTA (one thread per column) and reused by all voxels of the column in the
//    brick — chi1 does not depend on x3.
//  * The row walk of every voxel runs in float32 relative to the voxel centre
//    zc and to the integer detector row m_c nearest to the projection of zc.
//    Only the anchor chi2(zc) is formed in float64 (exact mode); every other
//    quantity is O(voxel) in magnitude, so float32 keeps ~1e-7 relative
//    accuracy where the reference's own float path (world coordinates) loses
//    ~1e-5. This is what lets the exact mode meet the
//    1e-5 rel-L2 bar at float32 throughput.
#pragma once

#include <math.h>

#include "common.cuh"

namespace cvpb {

template <typename G> struct V2 {
    G x, y;
};

template <typename G> struct Poly {
    V2<G> v[8];
    int n;
};

template <typename G> struct HalfPlane {
    G nx, ny, off;
};

template <typename G> __device__ __forceinline__ G gabs(G x) { return x < G(0) ? -x : x; }

// View constants in geometry precision G (ViewCtx<T>, cvp.cpp:26-56).
template <typename G> struct ViewG {
    G sx, sy, w1x, w1y, w3x, w3y;
    double w1x_d, w1y_d, w3x_d, w3y_d, sx_d, sy_d;
};

template <typename G> __device__ __forceinline__ ViewG<G> load_view_g(const ViewConst& vc) {
    ViewG<G> g;
    g.w1x_d = vc.w1x;
    g.w1y_d = vc.w1y;
    g.w3x_d = vc.w3x;
    g.w3y_d = vc.w3y;
    g.sx_d = vc.sx;
    g.sy_d = vc.sy;
    g.sx = G(vc.sx);
    g.sy = G(vc.sy);
    g.w1x = G(vc.w1x);
    g.w1y = G(vc.w1y);
    g.w3x = G(vc.w3x);
    g.w3y = G(vc.w3y);
    return g;
}

// Pre-image of chi1 <= c: built in float64 and narrowed afterwards, exactly as
// the reference does even in Single mode (cvp.cpp:65-69, polygon.hpp:18-22).
template <typename G>
__device__ __forceinline__ HalfPlane<G> chi1_le(const ViewG<G>& v, double c) {
    double nx = v.w1x_d - c * v.w3x_d;
    double ny = v.w1y_d - c * v.w3y_d;
    double off = nx * v.sx_d + ny * v.sy_d;
    double inv = 1.0 / sqrt(nx * nx + ny * ny);
    return {G(nx * inv), G(ny * inv), G(off * inv)};
}

template <typename G> __device__ __forceinline__ G poly_area(const Poly<G>& p) {
    G twice = G(0);
    for (int i = 0; i < p.n; ++i) {
        int j = (i + 1 == p.n) ? 0 : i + 1;
        twice += p.v[i].x * p.v[j].y - p.v[i].y * p.v[j].x;
    }
    return twice * G(0.5);
}

// Sutherland–Hodgman clip by a closed half-plane, boundary vertices kept,
// vertices merged at 1e-12*scale and slivers (< 1e-14*scale^2) dropped
// (polygon.hpp:101-155).
template <typename G>
__device__ __forceinline__ void poly_clip(const Poly<G>& p, const HalfPlane<G>& h, Poly<G>& out) {
    out.n = 0;
    const int n = p.n;
    if (n == 0) return;
    G dist[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (i < n) dist[i] = h.nx * p.v[i].x + h.ny * p.v[i].y - h.off;
    V2<G> raw[9];
    int m = 0;
    for (int i = 0; i < n; ++i) {
        const int j = (i + 1 == n) ? 0 : i + 1;
        const G di = dist[i], dj = dist[j];
        if (di <= G(0)) raw[m++] = p.v[i];
        if ((di < G(0) && dj > G(0)) || (di > G(0) && dj < G(0))) {
            const G t = di / (di - dj);
            raw[m++] = {p.v[i].x + (p.v[j].x - p.v[i].x) * t, p.v[i].y + (p.v[j].y - p.v[i].y) * t};
        }
    }
    if (m < 3) return;
    G s = G(0);
    for (int i = 0; i < m; ++i) s = fmax(s, fmax(gabs(raw[i].x), gabs(raw[i].y)));
    const G eps = G(1e-12) * s;
    out.v[0] = raw[0];
    out.n = 1;
    for (int i = 1; i < m; ++i) {
        const G dx = raw[i].x - out.v[out.n - 1].x, dy = raw[i].y - out.v[out.n - 1].y;
        if ((gabs(dx) > eps || gabs(dy) > eps) && out.n < 8) out.v[out.n++] = raw[i];
    }
    if (out.n >= 2) {
        const G dx = out.v[out.n - 1].x - out.v[0].x, dy = out.v[out.n - 1].y - out.v[0].y;
        if (gabs(dx) <= eps && gabs(dy) <= eps) out.n -= 1;
    }
    if (out.n < 3) {
        out.n = 0;
        return;
    }
    G sc = G(0);
    for (int i = 0; i < out.n; ++i) sc = fmax(sc, fmax(gabs(out.v[i].x), gabs(out.v[i].y)));
    if (poly_area(out) < G(1e-14) * sc * sc) out.n = 0;
}

// One column cut reduced to what the float32 row walk needs.
struct CutRec {
    int n;         // detector column
    double q;      // f/(b2 d0): chi2 per mm of z at the centroid depth (anchor slope)
    float g;       // b2 d0 / f: mm of z per detector row at the centroid depth
    float A;       // cut area [mm^2]
    float rho2;    // |centroid - source_xy|^2
    float bh;      // (b2/f) * hw: beta per row offset
    float halfw;   // rectangle half-width (elevation correction)
    float dd;      // |hw| * halfw: depth spread of the rectangle
    float d0;      // depth at the centroid
};

// Visits the column cuts of voxel column (i, j) in order of increasing
// detector column n (BandCutter + compute_cuts + fill_cut_info,
// cvp.cpp:73-157). Calls on_cut(const CutRec&) for each cut with positive
// area and returns the number of such cuts; returns -1 when the base reaches
// the source plane (the reference throws std::runtime_error, cvp.cpp:82-84)
// and -2 on a degenerate centroid (std::domain_error, polygon.hpp:94).
// Also reports |bc - s|^2 (VoxelCenter radius, cvp.cpp:338-339).
template <typename G, class OnCut>
__device__ int visit_column_cuts(const ViewConst& vc, const ViewG<G>& v, const Scene& sc, int i,
                                 int j, bool clamp_cols, bool need_width, float* rho2_center,
                                 OnCut&& on_cut) {
    const double bcx = sc.minx + (i + 0.5) * sc.a1;
    const double bcy = sc.miny + (j + 0.5) * sc.a2;
    Poly<G> base;
    base.n = 4;
    const G lx = G(bcx - 0.5 * sc.a1), ly = G(bcy - 0.5 * sc.a2);
    const G hx = G(bcx + 0.5 * sc.a1), hy = G(bcy + 0.5 * sc.a2);
    base.v[0] = {lx, ly};
    base.v[1] = {hx, ly};
    base.v[2] = {hx, hy};
    base.v[3] = {lx, hy};
    {
        const G rx = G(bcx) - v.sx, ry = G(bcy) - v.sy;
        *rho2_center = float(rx * rx + ry * ry);
    }
    G cmin = G(INFINITY), cmax = -G(INFINITY);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const G px = base.v[c].x - v.sx, py = base.v[c].y - v.sy;
        const G depth = v.w3x * px + v.w3y * py;
        if (!(depth > G(0))) return -1;
        const G chi1 = (v.w1x * px + v.w1y * py) / depth;
        cmin = fmin(cmin, chi1);
        cmax = fmax(cmax, chi1);
    }
    const int n_lo = int(ceil(double(cmin) - 0.5));
    const int n_hi = int(floor(double(cmax) + 0.5));
    const bool single = (n_lo == n_hi);
    int lo = n_lo, hi = n_hi;
    if (clamp_cols) {
        lo = max(lo, 0);
        hi = min(hi, sc.cols - 1);
    }
    int count = 0;
    Poly<G> tmp, piece;
    for (int n = lo; n <= hi; ++n) {
        const Poly<G>* pc;
        if (single && n == n_lo) {
            pc = &base;
        } else {
            // band_cut = clip(clip(square, upper), complement(lower)) (polygon.hpp:160-164)
            poly_clip(base, chi1_le(v, n + 0.5), tmp);
            HalfPlane<G> lower = chi1_le(v, n - 0.5);
            lower.nx = -lower.nx;
            lower.ny = -lower.ny;
            lower.off = -lower.off;
            poly_clip(tmp, lower, piece);
            pc = &piece;
        }
        const Poly<G>& P = *pc;
        if (P.n == 0) continue;
        // fill_cut_info (cvp.cpp:111-136)
        G twice = G(0), ax = G(0), ay = G(0);
        for (int a = 0; a < P.n; ++a) {
            const int b = (a + 1 == P.n) ? 0 : a + 1;
            const G cr = P.v[a].x * P.v[b].y - P.v[a].y * P.v[b].x;
            twice += cr;
            ax += (P.v[a].x + P.v[b].x) * cr;
            ay += (P.v[a].y + P.v[b].y) * cr;
        }
        const G area = twice * G(0.5);
        if (!(gabs(twice) > G(0))) return -2;
        const G cmx = ax / (G(3) * twice), cmy = ay / (G(3) * twice);
        const G rx = cmx - v.sx, ry = cmy - v.sy;
        const G rho2 = rx * rx + ry * ry;
        const G rho = sqrt(rho2);
        const G d0 = v.w3x * rx + v.w3y * ry;
        const G hw = d0 / rho;
        G halfw = G(0);
        if (need_width) {
            const G phx = -ry / rho, phy = rx / rho;
            G plo = G(INFINITY), phi = -G(INFINITY);
            for (int a = 0; a < P.n; ++a) {
                const G t = phx * P.v[a].x + phy * P.v[a].y;
                plo = fmin(plo, t);
                phi = fmax(phi, t);
            }
            const G ext = phi - plo;
            if (ext > G(0)) halfw = area / ext * G(0.5);
        }
        if (!(area > G(0))) continue;
        CutRec r;
        r.n = n;
        r.q = vc.f_over_b2 / double(d0);
        r.g = float(vc.b2_over_f * double(d0));
        r.A = float(area);
        r.rho2 = float(rho2);
        r.bh = float(vc.b2_over_f * double(hw));
        r.halfw = float(halfw);
        r.dd = float(gabs(hw) * halfw);
        r.d0 = float(d0);
        on_cut(r);
        ++count;
    }
    return count;
}

__device__ __forceinline__ float clampf(float x, float lo, float hi) {
    return fminf(fmaxf(x, lo), hi);
}

// Mean of clamp(alpha + beta*xi, -h, h) over xi in [-halfw, halfw]
// (clamp_mean, cvp.cpp:161-175), in voxel-local coordinates (z_lo = -h,
// z_hi = h).
__device__ __forceinline__ float clamp_mean_local(float alpha, float beta, float halfw, float h) {
    const float spread = fabsf(beta) * halfw;
    if (!(spread > 0.f)) return clampf(alpha, -h, h);
    const float glo = alpha - spread, ghi = alpha + spread;
    if (glo >= -h && ghi <= h) return alpha;
    if (ghi <= -h) return -h;
    if (glo >= h) return h;
    const float ca = clampf(glo, -h, h), cb = clampf(ghi, -h, h);
    const float below = fmaxf(0.f, fminf(ghi, -h) - glo);
    const float above = fmaxf(0.f, ghi - fmaxf(glo, h));
    const float integral = -h * below + 0.5f * (cb - ca) * (cb + ca) + h * above;
    return integral / (ghi - glo);
}

// Row walk of one voxel against one column cut (visit_rows, cvp.cpp:180-235)
// in voxel-local float32. ck = chi2 of the voxel centre at the centroid depth,
// dz = zc - s3, h = a3/2. emit(m, n, volume, inv_r2).
template <bool CLAMP, class Emit>
__device__ __forceinline__ void walk_rows(const CutRec& c, double ck, double pp2, float fb2,
                                          float dz, float h, bool corrected, bool per_row_r,
                                          float inv_r2_fixed, int rows, Emit&& emit) {
    const double mcd = rint(ck);
    const int mc = int(mcd);
    const float u = float(ck - mcd);    // |u| <= 0.5
    const float pm = float(pp2 - mcd);  // pp2 - m_c
    // Row range from the four (z, depth) corners (cvp.cpp:183-201):
    // chi2(zc+zl, d0+s*dd) - ck = fb2 * (s*dz*dd - zl*d0) / (d0*(d0 + s*dd)).
    float lo_off, hi_off;
    {
        const float d0 = c.d0;
        if (corrected) {
            const float dd = c.dd;
            const float ip = fb2 / (d0 * (d0 + dd)), im = fb2 / (d0 * (d0 - dd));
            const float a = (dz * dd - h * d0) * ip, b = (dz * dd + h * d0) * ip;
            const float e = (-dz * dd - h * d0) * im, f = (-dz * dd + h * d0) * im;
            lo_off = fminf(fminf(a, b), fminf(e, f));
            hi_off = fmaxf(fmaxf(a, b), fmaxf(e, f));
        } else {
            const float t = h * fb2 / d0;
            lo_off = -t;
            hi_off = t;
        }
    }
    int m_first = mc + int(ceilf(u + lo_off - 0.5f));
    int m_last = mc + int(floorf(u + hi_off + 0.5f));
    if (CLAMP) {
        m_first = max(m_first, 0);
        m_last = min(m_last, rows - 1);
    }
    if (m_first > m_last) return;
    // boundary chi_b = m - 0.5 in local units e = chi_b - m_c
    float e = float(m_first - mc) - 0.5f;
    float a_top = c.g * (u - e);
    float plain_top = clampf(a_top, -h, h);
    float t_top = corrected ? clamp_mean_local(a_top, (pm - e) * c.bh, c.halfw, h) : plain_top;
    for (int m = m_first; m <= m_last; ++m) {
        e += 1.f;
        const float a_bot = c.g * (u - e);
        const float plain_bot = clampf(a_bot, -h, h);
        const float t_bot =
            corrected ? clamp_mean_local(a_bot, (pm - e) * c.bh, c.halfw, h) : plain_bot;
        const float share = t_top - t_bot;
        if (share > 0.f) {
            float inv_r2 = inv_r2_fixed;
            if (per_row_r) {
                const float zr = dz + 0.5f * (plain_top + plain_bot);
                inv_r2 = 1.f / (c.rho2 + zr * zr);
            }
            emit(m, c.n, c.A * share, inv_r2);
        }
        t_top = t_bot;
        plain_top = plain_bot;
    }
}

// Anchor chi2 of the voxel centre at the cut's centroid depth: float64 in
// exact mode, float32 in relaxed mode (reference Single semantics).
template <bool EXACT>
__device__ __forceinline__ double voxel_anchor(double pp2, double dz64, float dz, const CutRec& c) {
    if (EXACT) return fma(-dz64, c.q, pp2);
    const float ck = float(pp2) - dz * float(c.q);
    return double(ck);
}

}  // namespace cvpb
