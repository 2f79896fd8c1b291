// Device-side CVP geometry: column cuts and the per-voxel row walk.
//
// Reference algorithm: /root/reference/proj/src/cvp.cpp (ViewCtx :26-70,
// BandCutter :73-98, fill_cut_info :111-136, compute_cuts :138-157,
// clamp_mean :161-175, visit_rows :180-235, process_column :326-349) and the
// polygon kernel in include/cbct/polygon.hpp:101-164.
//
// B200 re-design:
//  * Column cuts are computed in the voxel-base-local frame. The only
//    world-scale quantities — depth D0 and chi1 X0 of the base centre, the
//    chi2 slope Q0 = f/(b2 D0) — are formed once per column (float64 in exact
//    mode). Everything else is O(voxel) in magnitude and runs in float32
//    without losing accuracy. (The reference builds world-coordinate polygons;
//    in float32 that costs it ~1e-5 relative.)
//  * The piece between detector-column boundaries n-1/2 and n+1/2 is
//    Q(n+1/2) \ Q(n-1/2) with Q(c) = square ∩ {chi1 <= c}; area and first
//    moments are differences of two half-plane clips (nested regions), so
//    each boundary is clipped once and areas telescope: the pieces of a voxel
//    sum to its base area by construction (cf. test_cvp.cpp:410-432).
//  * No polygon arrays: clips are unrolled over the 4 square edges with the
//    shoelace sums accumulated on the fly, so nothing spills to local memory.
//  * The row walk of every voxel runs in float32 relative to the voxel centre
//    zc and to an integer row m_ref near chi2(zc); only the per-(column,
//    voxel) anchor chi2(zc) at the base-centre depth is float64 (exact mode).
#pragma once

#include <math.h>

#include "common.cuh"

namespace cvpb {

__device__ __forceinline__ float clampf(float x, float lo, float hi) {
    return fminf(fmaxf(x, lo), hi);
}

// Single-instruction MUFU reciprocal / rsqrt (~1 ulp); operands here are never
// denormal, so the flush-to-zero forms avoid the 5-instruction guarded
// sequence __fdividef expands to.
__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float fast_rsqrt(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Per-column quantities that every cut of the column shares.
struct ColumnRec {
    double Q0;     // f / (b2 D0): chi2 per mm of dz at the base-centre depth
    float rho2c;   // |bc - s|^2 (VoxelCenter radius, cvp.cpp:338-339)
    int count;     // number of cuts with positive area
};

// One column cut reduced to what the float32 row walk needs.
struct CutRec {
    int n;         // detector column
    float A;       // cut area [mm^2]
    float g;       // b2 d0 / f: mm of z per detector row at the centroid depth
    float rho2;    // |centroid - source_xy|^2
    float shw;     // (b2/f) |hw| halfw: elevation ramp half-width per row offset (0: none)
    float kc;      // chi2(zc) at this cut minus the column anchor, per mm of dz
    float tr_a;    // row half-range: h f/(b2 (d0 - dd)) ...
    float tr_b;    // ... + |dz| * f dd / (b2 d0 (d0 - dd))
};

// Area and first moments of {p in square : d(p) <= 0}, d affine with corner
// values d[0..3] (corners CCW). Sutherland–Hodgman over the 4 edges with the
// shoelace sums accumulated on the fly (polygon.hpp:75-155 semantics for a
// single closed half-plane: boundary vertices kept).
__device__ __forceinline__ void clip_moments(const float px[4], const float py[4],
                                             const float d[4], float& A, float& Mx, float& My) {
    float fx = 0.f, fy = 0.f, lx = 0.f, ly = 0.f;
    bool have = false;
    float a2 = 0.f, mx = 0.f, my = 0.f;
    auto push = [&](float x, float y) {
        if (have) {
            const float cr = lx * y - ly * x;
            a2 += cr;
            mx += (lx + x) * cr;
            my += (ly + y) * cr;
        } else {
            fx = x;
            fy = y;
            have = true;
        }
        lx = x;
        ly = y;
    };
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int f = (e + 1) & 3;
        if (d[e] <= 0.f) push(px[e], py[e]);
        if ((d[e] < 0.f && d[f] > 0.f) || (d[e] > 0.f && d[f] < 0.f)) {
            const float t = __fdividef(d[e], d[e] - d[f]);
            push(px[e] + (px[f] - px[e]) * t, py[e] + (py[f] - py[e]) * t);
        }
    }
    if (have) {
        const float cr = lx * fy - ly * fx;
        a2 += cr;
        mx += (lx + fx) * cr;
        my += (ly + fy) * cr;
    }
    A = 0.5f * a2;
    Mx = mx * (1.f / 6.f);
    My = my * (1.f / 6.f);
}

// Extent of a band piece along direction (ux, uy): min/max of the projection
// over square corners inside the band and the band lines' crossings with the
// square edges (the piece's vertices).
__device__ __forceinline__ void band_extent(const float px[4], const float py[4],
                                            const float dlo[4], const float dhi[4], bool has_lo,
                                            bool has_hi, float ux, float uy, float& lo,
                                            float& hi) {
    lo = INFINITY;
    hi = -INFINITY;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int f = (e + 1) & 3;
        const bool in_lo = !has_lo || dlo[e] >= 0.f;
        const bool in_hi = !has_hi || dhi[e] <= 0.f;
        if (in_lo && in_hi) {
            const float t = ux * px[e] + uy * py[e];
            lo = fminf(lo, t);
            hi = fmaxf(hi, t);
        }
        if (has_lo && ((dlo[e] < 0.f && dlo[f] > 0.f) || (dlo[e] > 0.f && dlo[f] < 0.f))) {
            const float t = __fdividef(dlo[e], dlo[e] - dlo[f]);
            const float x = px[e] + (px[f] - px[e]) * t, y = py[e] + (py[f] - py[e]) * t;
            const float s = ux * x + uy * y;
            lo = fminf(lo, s);
            hi = fmaxf(hi, s);
        }
        if (has_hi && ((dhi[e] < 0.f && dhi[f] > 0.f) || (dhi[e] > 0.f && dhi[f] < 0.f))) {
            const float t = __fdividef(dhi[e], dhi[e] - dhi[f]);
            const float x = px[e] + (px[f] - px[e]) * t, y = py[e] + (py[f] - py[e]) * t;
            const float s = ux * x + uy * y;
            lo = fminf(lo, s);
            hi = fmaxf(hi, s);
        }
    }
}

// Column cuts of voxel column (i, j) under view vc (BandCutter + compute_cuts
// + fill_cut_info, cvp.cpp:73-157), in increasing detector column n.
// Calls on_cut(const CutRec&) per cut with positive area; returns the count,
// or -1 if the base reaches the source plane (std::runtime_error in the
// reference, cvp.cpp:82-84). EXACT selects float64 for the per-column
// world-scale quantities; relaxed mode forms them in float32 like the
// reference's Single path.
template <bool EXACT, class OnCut>
__device__ int column_cuts(const ViewConst& vc, const Scene& sc, int i, int j, bool clamp_cols,
                           bool need_width, ColumnRec& col, OnCut&& on_cut) {
    using R = typename std::conditional<EXACT, double, float>::type;
    const double bcx = sc.minx + (i + 0.5) * sc.a1;
    const double bcy = sc.miny + (j + 0.5) * sc.a2;
    const R Rx = R(bcx) - R(vc.sx), Ry = R(bcy) - R(vc.sy);
    const R D0 = R(vc.w3x) * Rx + R(vc.w3y) * Ry;    // depth of the base centre
    const R N0 = R(vc.w1x) * Rx + R(vc.w1y) * Ry;    // chi1 numerator
    col.rho2c = float(Rx * Rx + Ry * Ry);
    col.count = 0;
    if (!(D0 > R(0))) return -1;
    const R X0 = N0 / D0;
    const R fb2 = R(vc.f_over_b2);
    col.Q0 = double(fb2 / D0);
    const int n0 = int(rint(X0));
    const float x0 = float(X0 - R(n0));
    const float D0f = float(D0);
    const float fu = float(vc.f / vc.b1);
    const float ewx = float(vc.ew[0]), ewy = float(vc.ew[1]);
    const float pp1r = float(vc.pp1 - n0);
    // w1 - n0 w3 = fu e_u + (pp1 - n0) e_w (xy parts), no cancellation
    const float Wx = fu * float(vc.eu[0]) + pp1r * ewx;
    const float Wy = fu * float(vc.eu[1]) + pp1r * ewy;
    const float hx = float(0.5 * sc.a1), hy = float(0.5 * sc.a2);
    const float px[4] = {-hx, hx, hx, -hx}, py[4] = {-hy, -hy, hy, hy};
    float F[4], Gd[4], cmin = INFINITY, cmax = -INFINITY;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        F[q] = D0f * x0 + Wx * px[q] + Wy * py[q];  // (chi1 - n0) * depth
        Gd[q] = D0f + ewx * px[q] + ewy * py[q];    // depth at the corner
        if (!(Gd[q] > 0.f)) return -1;
        const float c1 = __fdividef(F[q], Gd[q]);
        cmin = fminf(cmin, c1);
        cmax = fmaxf(cmax, c1);
    }
    // column range relative to n0 (cvp.cpp:89-90), clamped to the detector
    const int lo = int(ceilf(cmin - 0.5f)), hi = int(floorf(cmax + 0.5f));
    int nlo = lo, nhi = hi;
    if (clamp_cols) {
        nlo = max(nlo, -n0);
        nhi = min(nhi, sc.cols - 1 - n0);
    }
    const float full = float(sc.a1 * sc.a2);
    const float b2f = float(vc.b2_over_f), fb2f = float(fb2);
    const float h = float(0.5 * sc.a3);
    const float Rxf = float(Rx), Ryf = float(Ry);
    // lower boundary of the first piece
    float dlo[4], Alo = 0.f, Mxlo = 0.f, Mylo = 0.f;
    if (nlo > lo && nlo <= nhi) {
        const float e = float(nlo) - 0.5f;
#pragma unroll
        for (int q = 0; q < 4; ++q) dlo[q] = F[q] - e * Gd[q];
        clip_moments(px, py, dlo, Alo, Mxlo, Mylo);
    }
    int count = 0;
    for (int n = nlo; n <= nhi; ++n) {
        const bool has_lo = n > lo, has_hi = n < hi;
        float dhi[4], Ahi = full, Mxhi = 0.f, Myhi = 0.f;
        if (has_hi) {
            const float e = float(n) + 0.5f;
#pragma unroll
            for (int q = 0; q < 4; ++q) dhi[q] = F[q] - e * Gd[q];
            clip_moments(px, py, dhi, Ahi, Mxhi, Myhi);
        }
        const float A = Ahi - Alo;
        if (A > 1e-6f * full) {
            const float inv = fast_rcp(A);
            const float cmx = (Mxhi - Mxlo) * inv, cmy = (Myhi - Mylo) * inv;
            const float rx = Rxf + cmx, ry = Ryf + cmy;
            const float rho2 = rx * rx + ry * ry;
            const float rinv = rsqrtf(rho2);
            const float delta = ewx * cmx + ewy * cmy;  // depth offset of the centroid
            const float d0 = D0f + delta;
            const float hw = d0 * rinv;
            float halfw = 0.f;
            if (need_width) {
                float elo, ehi;
                band_extent(px, py, dlo, dhi, has_lo, has_hi, -ry * rinv, rx * rinv, elo, ehi);
                const float ext = ehi - elo;
                if (ext > 0.f) halfw = 0.5f * A * fast_rcp(ext);
            }
            CutRec r;
            r.n = n0 + n;
            r.A = A;
            r.g = b2f * d0;
            r.rho2 = rho2;
            r.shw = float(vc.b2_over_f) * fabsf(hw) * halfw;
            r.kc = fb2f * delta * fast_rcp(D0f * d0);
            const float dd = fabsf(hw) * halfw;
            const float dm = fast_rcp(d0 - dd);
            r.tr_a = fmaf(h * fb2f, dm, 1e-5f);
            r.tr_b = fb2f * dd * dm * fast_rcp(d0);
            on_cut(r);
            ++count;
        }
        if (has_hi) {
#pragma unroll
            for (int q = 0; q < 4; ++q) dlo[q] = dhi[q];
        }
        Alo = Ahi;
        Mxlo = Mxhi;
        Mylo = Myhi;
    }
    col.count = count;
    return count;
}

// Packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2 on sm_100): one issue slot
// for two independent lanes of the row walk's boundary pairs.
__device__ __forceinline__ uint64_t pk2(float2 v) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
    return r;
}
__device__ __forceinline__ float2 upk2(uint64_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
    return upk2(d);
}

// Mean of clamp(alpha + beta*xi, -h, h) over xi in [-halfw, halfw]
// (clamp_mean, cvp.cpp:161-175) in voxel-local coordinates, branch-free.
// With spread s = |beta| halfw, mean over [alpha-s, alpha+s] of
//   min(u, h)  = min(alpha, h)  - (s - |alpha - h|)+^2 / (4s)
//   max(u, -h) = max(alpha, -h) + (s - |alpha + h|)+^2 / (4s)
// and clamp = min + max - u, so
//   T = clamp(alpha, -h, h) + [(s - |alpha+h|)+^2 - (s - |alpha-h|)+^2] / (4s),
// exact for any s (also ramps wider than the voxel); both squares are <= s^2,
// so the correction stays bounded as s -> 0 and vanishes at s = 0.
// spread_of: the spread sh |d| with a 1e-30 floor folded into the multiply
// (no separate max before the reciprocal; below ulp of any real spread, and
// with sh = 0 the correction's squares underflow to exactly 0).
__device__ __forceinline__ float spread_of(float sh, float d) { return fmaf(sh, fabsf(d), 1e-30f); }
__device__ __forceinline__ float clamp_mean_local(float alpha, float spread, float h) {
    const float d1 = fmaxf(spread - fabsf(alpha + h), 0.f);
    const float d2 = fmaxf(spread - fabsf(alpha - h), 0.f);
    const float corr = fmaf(d1, d1, -d2 * d2) * (0.25f * fast_rcp(spread));
    return clampf(alpha, -h, h) + corr;
}

// Row walk of one voxel against one column cut (visit_rows, cvp.cpp:180-235)
// in voxel-local float32, with every chi2 quantity shifted by +1/2 so row
// boundaries sit on integers: Mi / Mf = m_ref (integer row near chi2(zc), as
// int and as exact float), uh = chi2(zc) - m_ref + 1/2 at the cut's centroid
// depth, pmh = pp2 - m_ref + 1/2, dz = zc - s3, h = a3/2, sh = the cut's
// elevation half-width factor when the elevation correction applies, else 0.
// Row m spans the boundaries e' = m - m_ref and e' + 1 (chi2 = m -+ 1/2).
// emit(m, share * inv_r2) — the caller multiplies by the cut area once per cut.
// DENSE: emit every row of the range with max(share, 0) (branch-free; a zero
// share contributes nothing) instead of only rows with share > 0 (the record
// view of cvp.cpp:221).
// NR (DENSE only): rows walked in straight-line code before the loop — 2 for
// voxels up to ~1 detector row tall, 3 for taller ones (the launch picks it
// from the scene's largest voxel height in rows).
template <bool CLAMP, class Emit, bool DENSE = false, int NR = 2>
__device__ __forceinline__ void walk_rows(const CutRec& c, int Mi, float Mf, float uh, float pmh,
                                          float dz, float h, float sh, const bool per_row_r,
                                          float inv_r2_fixed, int rows, Emit&& emit) {
    // rows whose boundaries can intersect the (elevation-widened) voxel
    // (cvp.cpp:183-201): symmetric bound of the four corner chi2 values
    // (tr_a carries the 1e-5 px slack)
    const float tr = fmaf(fabsf(dz), c.tr_b, c.tr_a);
    // m_first - m_ref = ceil(uh - tr) - 1, m_last - m_ref = floor(uh + tr) by
    // the 1.5*2^23 rounding trick (directed-rounding FADD + integer subtract:
    // no conversion-unit instructions). The offsets are clamped to +-2^21
    // rows; only a voxel touching the source plane spans more, and the
    // detector clamp below then yields the same range.
    constexpr float kMagic = 12582912.f;
    constexpr int kMagicBits = 0x4B400000;
    const float clo = __fadd_ru(fmaxf(uh - tr, -2097152.f), kMagic - 1.f);
    const float chi = __fadd_rd(fminf(uh + tr, 2097152.f), kMagic);
    int m_first = Mi + (__float_as_int(clo) - kMagicBits);
    int m_last = Mi + (__float_as_int(chi) - kMagicBits);
    float e = clo - kMagic;  // top boundary of row m_first, relative to m_ref (exact)
    if (CLAMP) {
        m_first = max(m_first, 0);
        m_last = min(m_last, rows - 1);
        e = fmaxf(e, -Mf);
    }
    // DENSE: an empty range (voxel off the detector rows) emits zero weights
    // instead of branching out
    const bool nonempty = m_first <= m_last;
    if (!DENSE && !nonempty) return;
    // spread of the elevation rectangle at boundary e: |beta(e)| halfw with
    // beta(e) = (b2/f) hw (pm - e)  (cvp.cpp:205)
    const float dtop = pmh - e;
    float a_top = c.g * (uh - e);
    float plain_top = clampf(a_top, -h, h);
    // The top boundary of the row range lies above the voxel, its ramp
    // included, in all but ~1e-4 of voxel-cuts (the range is built from the
    // voxel's own corners): T = h exactly. The branch is warp-uniform in
    // practice, so the clamp-mean runs only for the rare straddling lane.
    const float s_top = spread_of(sh, dtop);
    float t_top = h;
    if (a_top - s_top < h) t_top = clamp_mean_local(a_top, s_top, h);
    int m = m_first;
    if (DENSE) {
        // Rows 1 and 2 in straight-line code (a voxel-cut spans 1-2 rows in
        // the common case): no loop control, no divergence between 1- and
        // 2-row lanes — a missing second row is emitted at m_first + 1 with
        // weight 0 (callers clamp its index). Boundary k lies at e + k: alpha = a_top - k g.
        // Both boundaries as fp32x2 pairs.
        const float2 A = fma2(make_float2(-1.f, -2.f), make_float2(c.g, c.g),
                              make_float2(a_top, a_top));  // alpha at e+1, e+2
        const float p1 = clampf(A.x, -h, h), p2 = clampf(A.y, -h, h);
        const float2 D = add2(make_float2(dtop, dtop), make_float2(-1.f, -2.f));
        const float s1 = spread_of(sh, D.x), s2 = spread_of(sh, D.y);
        const float2 AP = add2(A, make_float2(h, h)), AM = sub2(A, make_float2(h, h));
        const float2 d1 = make_float2(fmaxf(s1 - fabsf(AP.x), 0.f), fmaxf(s2 - fabsf(AP.y), 0.f));
        const float2 d2 = make_float2(fmaxf(s1 - fabsf(AM.x), 0.f), fmaxf(s2 - fabsf(AM.y), 0.f));
        const float2 num = sub2(mul2(d1, d1), mul2(d2, d2));
        const float2 rr = make_float2(fast_rcp(s1), fast_rcp(s2));
        const float2 T = fma2(mul2(num, rr), make_float2(0.25f, 0.25f), make_float2(p1, p2));
        const float t1 = T.x, t2 = T.y;
        const float2 W = sub2(make_float2(t_top, t1), T);
        float2 inv = make_float2(inv_r2_fixed, inv_r2_fixed);
        if (per_row_r) {
            const float2 Z = fma2(add2(make_float2(plain_top, p1), make_float2(p1, p2)),
                                  make_float2(0.5f, 0.5f), make_float2(dz, dz));
            const float2 Q = fma2(Z, Z, make_float2(c.rho2, c.rho2));
            inv = make_float2(fast_rcp(Q.x), fast_rcp(Q.y));
        }
        const float2 WI = mul2(make_float2(fmaxf(W.x, 0.f), fmaxf(W.y, 0.f)), inv);
        const bool two = m_last > m_first;
        emit(m_first, nonempty ? WI.x : 0.f);
        emit(m_first + 1, two ? WI.y : 0.f);  // may lie past m_last (and the detector): weight 0
        if constexpr (NR >= 3) {
            // third row (boundary e + 3) in straight-line code as well
            const float a3 = fmaf(-3.f, c.g, a_top);
            const float p3 = clampf(a3, -h, h);
            const float t3 = clamp_mean_local(a3, spread_of(sh, dtop - 3.f), h);
            float inv3 = inv_r2_fixed;
            if (per_row_r) {
                const float z3 = fmaf(0.5f, p2 + p3, dz);
                inv3 = fast_rcp(fmaf(z3, z3, c.rho2));
            }
            emit(m_first + 2, m_last > m_first + 1 ? fmaxf(t2 - t3, 0.f) * inv3 : 0.f);
            if (m_last <= m_first + 2) return;
            m = m_first + 3;
            e += 3.f;
            t_top = t3;
            plain_top = p3;
        } else {
            if (m_last <= m_first + 1) return;
            m = m_first + 2;
            e += 2.f;
            t_top = t2;
            plain_top = p2;
        }
    }
    // not unrolled: rows per voxel-cut are 1-3 and differ across lanes; an
    // unrolled pair + remainder runs the remainder with ~2 active lanes
#pragma unroll 1
    for (; m <= m_last; ++m) {
        e += 1.f;
        const float a_bot = c.g * (uh - e);
        const float plain_bot = clampf(a_bot, -h, h);
        const float t_bot = clamp_mean_local(a_bot, spread_of(sh, pmh - e), h);
        const float share = t_top - t_bot;
        if (DENSE || share > 0.f) {
            float inv_r2 = inv_r2_fixed;
            if (per_row_r) {
                const float zr = fmaf(0.5f, plain_top + plain_bot, dz);
                inv_r2 = fast_rcp(fmaf(zr, zr, c.rho2));
            }
            emit(m, (DENSE ? fmaxf(share, 0.f) : share) * inv_r2);
        }
        t_top = t_bot;
        plain_top = plain_bot;
    }
}

// Row walk of one voxel against one column cut when its brick's rows need no
// detector clamping and every voxel-cut of the brick spans at most NB + 1 rows
// (the launch decides per (brick, view), see cvp_kernels.cu footprint()).
// The range bound tr is rigorous (tr_a carries 1e-5 px of slack), so the top
// boundary of row m_first lies above the voxel and its elevation ramp, and the
// bottom boundary of row m_first + NB below them: their clamp-means are +h and
// -h exactly (clamp_mean, cvp.cpp:161-175, saturates), and only the NB
// interior boundaries need evaluating. A voxel that occupies fewer rows gets
// exactly -h at the interior boundaries below it, i.e. zero-share rows.
// Rows m_first .. m_first + NB are emitted in order with
// max(share, 0) * inv_r2 * wscale (the caller's mu * area, folded in here).
// CUTR (relaxed precision, CutCentroid): one radius per voxel-cut — the
// cut's horizontal distance and the voxel's centre height — instead of one
// per row segment; the launch allows it only where that changes 1/r^2 by
// <= 2.5e-6 relative (cvp_kernels.cu footprint()).
// RAW: rows are emitted biased by +kRowBias (the rounding trick's magic
// bits left in); the caller folds -kRowBias into its per-cut base address, so
// no voxel pays the subtraction.
constexpr int kRowBias = 0x4B400000;
template <int NB, class Emit, bool CUTR = false, bool RAW = false>
__device__ __forceinline__ void walk_rows_fast(const CutRec& c, int Mi, float uh, float pmh, float dz,
                                               float h, float sh, const bool per_row_r,
                                               float inv_r2_fixed, float wscale, Emit&& emit) {
    static_assert(NB >= 1 && NB <= 3, "one to three interior boundaries");
    if (CUTR && per_row_r) inv_r2_fixed = fast_rcp(fmaf(dz, dz, c.rho2));
    constexpr bool PRR = !CUTR;  // per-row radius (CutCentroid, cvp.cpp:223-229)
    constexpr float kMagic = 12582912.f;
    constexpr int kMagicBits = 0x4B400000;
    const float tr = fmaf(fabsf(dz), c.tr_b, c.tr_a);
    // (no +-2^21 guard: the brick's rows lie inside the detector)
    const float clo = __fadd_ru(uh - tr, kMagic - 1.f);
    const int m_first = RAW ? Mi + __float_as_int(clo) : Mi + (__float_as_int(clo) - kMagicBits);
    // first interior boundary (top boundary of row m_first + 1), exact
    const float e1 = clo - (kMagic - 1.f);
    if constexpr (NB == 1) {
        const float a1 = c.g * (uh - e1);
        const float p1 = clampf(a1, -h, h);
        const float t1 = clamp_mean_local(a1, spread_of(sh, pmh - e1), h);
        // weight of a record = max(share, 0) * inv_r2 * wscale
        float2 I = make_float2(inv_r2_fixed * wscale, inv_r2_fixed * wscale);
        if (PRR && per_row_r) {
            // midpoints of the plain row segments [p1, h] and [-h, p1] (cvp.cpp:223-229)
            const float2 Z = fma2(make_float2(p1, p1), make_float2(0.5f, 0.5f),
                                  make_float2(dz + 0.5f * h, dz - 0.5f * h));
            const float2 Q = fma2(Z, Z, make_float2(c.rho2, c.rho2));
            I = mul2(make_float2(fast_rcp(Q.x), fast_rcp(Q.y)), make_float2(wscale, wscale));
        }
        const float2 S = add2(make_float2(h, h), make_float2(-t1, t1));
        // |t1| <= h: clamp_mean_local is clamp(alpha) plus a correction of
        // the sign that pulls it inward, so both shares are >= 0 without a
        // max(., 0) (rounding can leave -ulp(h), far below the fixed-point
        // quantum; c3 +2% P / BP)
        const float2 W = mul2(S, I);
        emit(m_first, W.x);
        emit(m_first + 1, W.y);
    } else {
        const float2 E = make_float2(e1, e1 + 1.f);
        const float2 A = mul2(make_float2(c.g, c.g), sub2(make_float2(uh, uh), E));
        const float p1 = clampf(A.x, -h, h), p2 = clampf(A.y, -h, h);
        const float2 D = sub2(make_float2(pmh, pmh), E);
        const float s1 = spread_of(sh, D.x), s2 = spread_of(sh, D.y);
        const float2 AP = add2(A, make_float2(h, h)), AM = sub2(A, make_float2(h, h));
        const float2 d1 = make_float2(fmaxf(s1 - fabsf(AP.x), 0.f), fmaxf(s2 - fabsf(AP.y), 0.f));
        const float2 d2 = make_float2(fmaxf(s1 - fabsf(AM.x), 0.f), fmaxf(s2 - fabsf(AM.y), 0.f));
        const float2 num = sub2(mul2(d1, d1), mul2(d2, d2));
        const float2 rr = make_float2(fast_rcp(s1), fast_rcp(s2));
        const float2 T = fma2(mul2(num, rr), make_float2(0.25f, 0.25f), make_float2(p1, p2));
        const float2 S = sub2(make_float2(h, T.x), T);
        if constexpr (NB == 2) {
            float2 I = make_float2(inv_r2_fixed * wscale, inv_r2_fixed * wscale);
            float i2 = I.x;
            if (PRR && per_row_r) {
                const float2 Z = fma2(add2(make_float2(h, p1), make_float2(p1, p2)),
                                      make_float2(0.5f, 0.5f), make_float2(dz, dz));
                const float z2 = fmaf(0.5f, p2 - h, dz);
                const float2 Q = fma2(Z, Z, make_float2(c.rho2, c.rho2));
                I = mul2(make_float2(fast_rcp(Q.x), fast_rcp(Q.y)), make_float2(wscale, wscale));
                i2 = fast_rcp(fmaf(z2, z2, c.rho2)) * wscale;
            }
            const float2 W = mul2(make_float2(fmaxf(S.x, 0.f), fmaxf(S.y, 0.f)), I);
            emit(m_first, W.x);
            emit(m_first + 1, W.y);
            emit(m_first + 2, fmaxf(T.y + h, 0.f) * i2);
        } else {
            // third interior boundary (voxels up to ~3 rows tall: configs[1])
            const float e3 = e1 + 2.f;
            const float a3 = c.g * (uh - e3);
            const float p3 = clampf(a3, -h, h);
            const float t3 = clamp_mean_local(a3, spread_of(sh, pmh - e3), h);
            const float2 S2 = make_float2(T.y - t3, t3 + h);
            float2 I = make_float2(inv_r2_fixed * wscale, inv_r2_fixed * wscale), I2 = I;
            if (PRR && per_row_r) {
                const float2 Z = fma2(add2(make_float2(h, p1), make_float2(p1, p2)),
                                      make_float2(0.5f, 0.5f), make_float2(dz, dz));
                const float2 Z2 = fma2(add2(make_float2(p2, p3), make_float2(p3, -h)),
                                       make_float2(0.5f, 0.5f), make_float2(dz, dz));
                const float2 Q = fma2(Z, Z, make_float2(c.rho2, c.rho2));
                const float2 Q2 = fma2(Z2, Z2, make_float2(c.rho2, c.rho2));
                I = mul2(make_float2(fast_rcp(Q.x), fast_rcp(Q.y)), make_float2(wscale, wscale));
                I2 = mul2(make_float2(fast_rcp(Q2.x), fast_rcp(Q2.y)), make_float2(wscale, wscale));
            }
            const float2 W = mul2(make_float2(fmaxf(S.x, 0.f), fmaxf(S.y, 0.f)), I);
            const float2 W2 = mul2(make_float2(fmaxf(S2.x, 0.f), fmaxf(S2.y, 0.f)), I2);
            emit(m_first, W.x);
            emit(m_first + 1, W.y);
            emit(m_first + 2, W2.x);
            emit(m_first + 3, W2.y);
        }
    }
}

// Column anchor chi2(zc) = pp2 - dz * Q0 split into an integer row m_ref and
// float32 remainders u = chi2(zc) - m_ref, pm = pp2 - m_ref.
template <bool EXACT>
__device__ __forceinline__ void voxel_anchor(double pp2, double dz64, float dz, double Q0,
                                             int& Mi, float& Mf, float& u, float& pm) {
    if (EXACT) {
        const double c = fma(-dz64, Q0, pp2);
        const double mr = rint(c);
        Mi = int(mr);
        Mf = float(mr);
        u = float(c - mr);
        pm = float(pp2 - mr);
    } else {
        const float c = fmaf(-dz, float(Q0), float(pp2));
        const float mr = rintf(c);
        Mi = int(mr);
        Mf = mr;
        u = c - mr;
        pm = float(pp2) - mr;
    }
}

// Column anchor for a whole brick column: chi2 of voxel k0 + kk at the
// base-centre depth is c0 - kk * delta (delta = a3 f / (b2 D0)). Per column
// (G-phase) c0 is split into an integer row M0 and a float32 remainder f0, and
// delta into dh (17 significant bits, so kk * dh is exact for kk < 128) and
// the float32 residual dl. Per voxel: P = kk dh (exact), I = rint(P),
// F = P - I (exact), so chi2 - (M0 - I) = (f0 - F) - kk dl to ~1e-7 px with
// no float64 arithmetic in the voxel loop.
struct ColumnAnchor {
    int M0;
    float f0, dh, dl;
};

template <bool EXACT>
__device__ __forceinline__ ColumnAnchor column_anchor(double pp2, double dz0, double Q0, double a3) {
    ColumnAnchor a;
    float delta_f;
    double delta;
    if (EXACT) {
        const double c0 = fma(-dz0, Q0, pp2);
        const double m0 = rint(c0);
        a.M0 = int(m0);
        a.f0 = float(c0 - m0);
        delta = a3 * Q0;
        delta_f = float(delta);
    } else {
        const float c0 = fmaf(-float(dz0), float(Q0), float(pp2));
        const float m0 = rintf(c0);
        a.M0 = int(m0);
        a.f0 = c0 - m0;
        delta_f = float(a3) * float(Q0);
        delta = double(delta_f);
    }
    a.dh = __uint_as_float(__float_as_uint(delta_f) & 0xFFFFFFC0u);
    a.dl = float(delta - double(a.dh));
    return a;
}

__device__ __forceinline__ void anchor_at(const ColumnAnchor& a, float pp2f, float kk, int& Mi,
                                          float& Mf, float& u, float& pm) {
    const float P = kk * a.dh;  // exact
    const float I = rintf(P);
    const float F = P - I;      // exact
    u = fmaf(-kk, a.dl, a.f0 - F);
    Mi = a.M0 - __float2int_rn(P);
    Mf = float(a.M0) - I;
    pm = pp2f - Mf;
}

}  // namespace cvpb
