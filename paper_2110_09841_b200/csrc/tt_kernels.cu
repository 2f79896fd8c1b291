// TT — separable trapezoid-footprint projector pair for sm_100a.
//
// The reference implementation has no TT code (SPEC.md:8 declares it out of
// scope; the paper only cites it). This follows the SF-TT
// model of Long, Fessler & Balter, "3D forward and back-projection for X-ray
// CT using separable footprints", IEEE TMI 29(11), 2010, restated from the
// published description (parity unpinned; validated by adjointness, footprint
// mass and accuracy against high-K Siddon, tests/test_tt_gpu.py):
//
//   P(m, n) = sum_j mu_j * a_j(m) * F1_j(n) * F2_j(m)
//
//   F1_j(n)  transaxial footprint: trapezoid through the detector-column
//            coordinates chi1 of the 4 base corners of voxel j (sorted
//            tau0..tau3, unit height), averaged over pixel column n;
//   F2_j(m)  axial footprint: trapezoid through chi2 of the voxel's z range
//            [z_lo, z_hi] at its nearest and farthest base-corner depths,
//            averaged over pixel row m;
//   a_j(m)   amplitude "A2": l_phi0 / cos theta(m) — the in-plane chord of the
//            voxel along its central ray, min(a1/|cos phi0|, a2/|sin phi0|),
//            stretched by the elevation of pixel row m seen at the voxel's
//            projected column ("A1" uses the voxel-centre elevation instead).
//
// Execution mirrors the CVP bricks (cvp_kernels.cu): one CTA per 16x8x64
// brick looping over views; per-column transaxial footprints computed once per
// view (float64 anchors); per-voxel axial footprint in voxel-local float32;
// forward accumulates into a shared detector tile, backward gathers from a
// shared copy of the image footprint.
#include <algorithm>

#include "cvp_device.cuh"  // ColumnAnchor / anchor_at: the voxel-local float32 chi2 anchor
#include "kernels.hpp"

namespace cvpb {

namespace {

#ifndef TT_BI
#define TT_BI 16
#endif
#ifndef TT_BJ
#define TT_BJ 8
#endif
constexpr int BI = TT_BI, BJ = TT_BJ, BK = 64;
constexpr int NCOL = BI * BJ;
#ifndef TT_NT
#define TT_NT 256
#endif
constexpr int NT = TT_NT;
constexpr int NWARP = NT / 32;
constexpr int NH = BK / 32;   // voxels per lane along x3
#ifndef TT_MINB
#define TT_MINB 4             // resident CTAs per SM (64 registers; measured faster than 3 at 80)
#endif
static_assert(NCOL < NT, "warps past the columns stage the tile");
static_assert(NT - BK > NCOL, "per-layer dz threads lie past the column and footprint threads");
constexpr int MAXN = 6;       // transaxial footprint width cached per column
constexpr int MUS = BK + 1;

struct TTParams {
    Scene sc;
    const ViewConst* views;
    const float* vol_in;
    float* vol_out;
    const float* proj_in;
    float* proj_out;
    int view_begin, view_count, views_per_group;
    int amplitude;            // 0 = A1, 1 = A2
    int tile_cap;
    int accumulate, atomic_out;
};

struct TTSmem {
    float f1[MAXN * NCOL];    // pixel-averaged transaxial footprint per column n0 + q
    int n0[NCOL], nn[NCOL];   // first detector column, count
    double Q0[NCOL];          // f / (b2 D0) at the base-centre depth (forward anchor)
    int4 anchor[NCOL];        // backward: ColumnAnchor {M0, f0, dh, dl} of the column's voxels
    float dz[BK];             // zc - s3 of the brick's voxel layers under this view
    float4 ax[NCOL];          // {dz coefficient at near depth, at far depth, h-term near, h-term far}
    float2 amp[NCOL];         // {l_phi0, 1/(u0^2 + f^2)}
    float vox[NCOL * MUS];
    int tile_m0, tile_n0, tile_rows, tile_cols, tile_stride, tile_ok;
    float mu_abs_max;         // forward: max |mu| over the brick
    float qscale;             // forward: fixed-point scale of this (brick, view)
    int nonfinite;            // forward: the brick holds a NaN / Inf attenuation
};

__device__ __forceinline__ void red_s32(int* a, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(a))),
                 "r"(v)
                 : "memory");
}

__device__ __forceinline__ float frcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Antiderivative of the unit-height trapezoid (t0 <= t1 <= t2 <= t3) at x,
// written without cancellation for narrow ramps.
__device__ __forceinline__ float trap_cdf(float x, float t0, float t1, float t2, float t3) {
    const float w1 = t1 - t0, w3 = t3 - t2;
    const float c1 = fminf(fmaxf(x, t0), t1);
    const float up = w1 > 0.f ? 0.5f * (c1 - t0) * (c1 - t0) * frcp(w1) : 0.f;
    const float mid = fminf(fmaxf(x, t1), t2) - t1;
    const float c3 = fminf(fmaxf(x, t2), t3);
    const float dn = w3 > 0.f ? 0.5f * (c3 - t2) * (t3 - t2 + t3 - c3) * frcp(w3) : 0.f;
    return up + mid + dn;
}

__device__ __forceinline__ void sort4(float& a, float& b, float& c, float& d) {
    float t;
    if (a > b) { t = a; a = b; b = t; }
    if (c > d) { t = c; c = d; d = t; }
    if (a > c) { t = a; a = c; c = t; }
    if (b > d) { t = b; b = d; d = t; }
    if (b > c) { t = b; b = c; c = t; }
}

// Transaxial footprint of column (i, j): writes up to MAXN pixel-averaged
// values starting at detector column *n_first; returns the count (may exceed
// MAXN for very wide footprints — the caller then recomputes).
__device__ int column_footprint(const ViewConst& vc, const Scene& sc, int i, int j, float* f1,
                                int& n_first, double& Q0, float4& axc, float2& amp, int amplitude) {
    const double bcx = sc.minx + (i + 0.5) * sc.a1, bcy = sc.miny + (j + 0.5) * sc.a2;
    const double Rx = bcx - vc.sx, Ry = bcy - vc.sy;
    const double D0 = vc.w3x * Rx + vc.w3y * Ry;
    const double X0 = (vc.w1x * Rx + vc.w1y * Ry) / D0;
    Q0 = vc.f_over_b2 / D0;
    const int nr = int(rint(X0));
    const float x0 = float(X0 - nr), D0f = float(D0);
    const float fu = float(vc.f / vc.b1);
    const float ewx = float(vc.ew[0]), ewy = float(vc.ew[1]);
    const float pp1r = float(vc.pp1 - nr);
    const float Wx = fu * float(vc.eu[0]) + pp1r * ewx, Wy = fu * float(vc.eu[1]) + pp1r * ewy;
    const float hx = float(0.5 * sc.a1), hy = float(0.5 * sc.a2);
    float tau[4], dep[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float px = (q == 1 || q == 2) ? hx : -hx, py = (q >= 2) ? hy : -hy;
        dep[q] = ewx * px + ewy * py;  // depth offset from D0
        tau[q] = (D0f * x0 + Wx * px + Wy * py) * frcp(D0f + dep[q]);
    }
    float t0 = tau[0], t1 = tau[1], t2 = tau[2], t3 = tau[3];
    sort4(t0, t1, t2, t3);
    const int lo = int(ceilf(t0 - 0.5f)), hi = int(floorf(t3 + 0.5f));
    int nlo = max(lo, -nr), nhi = min(hi, sc.cols - 1 - nr);
    int cnt = 0;
    float g_prev = trap_cdf(float(nlo) - 0.5f, t0, t1, t2, t3);
    for (int n = nlo; n <= nhi; ++n) {
        const float g = trap_cdf(float(n) + 0.5f, t0, t1, t2, t3);
        if (cnt < MAXN) f1[cnt] = g - g_prev;
        ++cnt;
        g_prev = g;
    }
    n_first = nr + nlo;
    // axial trapezoid coefficients at the nearest/farthest corner depths:
    // chi2(zc + zl, D0 + dl) - chi2_anchor = fb2 (dz dl - zl D0) / (D0 (D0 + dl))
    const float dn = fminf(fminf(dep[0], dep[1]), fminf(dep[2], dep[3]));
    const float df = fmaxf(fmaxf(dep[0], dep[1]), fmaxf(dep[2], dep[3]));
    const float fb2 = float(vc.f_over_b2);
    const float pn = fb2 * frcp(D0f * (D0f + dn)), pf = fb2 * frcp(D0f * (D0f + df));
    const float h = float(0.5 * sc.a3);
    axc = make_float4(dn * pn, df * pf, h * D0f * pn, h * D0f * pf);
    // amplitude: in-plane chord along the central ray, and the row-elevation term
    const float rx = float(Rx), ry = float(Ry);
    const float rinv = rsqrtf(rx * rx + ry * ry);
    const float cx = fabsf(rx) * rinv, cy = fabsf(ry) * rinv;
    const float lphi = fminf(cx > 0.f ? float(sc.a1) / cx : INFINITY, cy > 0.f ? float(sc.a2) / cy : INFINITY);
    const float u0 = float((X0 - vc.pp1) * vc.b1);
    amp = make_float2(lphi, 1.f / (u0 * u0 + float(vc.f * vc.f)));
    (void)amplitude;
    return cnt;
}

// Transaxial footprint of a column too wide for the cache (cnt > MAXN): the
// trapezoid in chi1 and the column range, re-derived per voxel.
struct WideColumn {
    float s0, s1, s2, s3;
    int nr, nlo, nhi;
};
__device__ WideColumn wide_column(const ViewConst& vc, const Scene& sc, int i, int j) {
    const double bcx = sc.minx + (i + 0.5) * sc.a1, bcy = sc.miny + (j + 0.5) * sc.a2;
    const double Rx = bcx - vc.sx, Ry = bcy - vc.sy;
    const double D0 = vc.w3x * Rx + vc.w3y * Ry;
    const double X0 = (vc.w1x * Rx + vc.w1y * Ry) / D0;
    WideColumn w;
    w.nr = int(rint(X0));
    const float x0 = float(X0 - w.nr), D0f = float(D0);
    const float fu = float(vc.f / vc.b1);
    const float ewx = float(vc.ew[0]), ewy = float(vc.ew[1]);
    const float pp1r = float(vc.pp1 - w.nr);
    const float Wx = fu * float(vc.eu[0]) + pp1r * ewx, Wy = fu * float(vc.eu[1]) + pp1r * ewy;
    const float hx = float(0.5 * sc.a1), hy = float(0.5 * sc.a2);
    float tau[4];
    for (int q = 0; q < 4; ++q) {
        const float px = (q == 1 || q == 2) ? hx : -hx, py = (q >= 2) ? hy : -hy;
        tau[q] = (D0f * x0 + Wx * px + Wy * py) / (D0f + ewx * px + ewy * py);
    }
    w.s0 = tau[0];
    w.s1 = tau[1];
    w.s2 = tau[2];
    w.s3 = tau[3];
    sort4(w.s0, w.s1, w.s2, w.s3);
    w.nlo = max(int(ceilf(w.s0 - 0.5f)), -w.nr);
    w.nhi = min(int(floorf(w.s3 + 0.5f)), sc.cols - 1 - w.nr);
    return w;
}

// One CTA per 16x8x64 brick looping over its views (the CVP brick layout,
// cvp_kernels.cu): warps 0-3 compute the per-column transaxial footprints
// while warps 4-7 bound the brick's detector footprint and stage the tile
// (named barrier); each lane then carries the voxels kk = lane, lane + 32 of
// a column through the axial walk.
// AMP2: amplitude A2 (per-row elevation) rather than A1 — a template flag so
// the unused one costs nothing in the row loop.
template <bool FWD, bool AMP2>
__global__ void __launch_bounds__(NT, TT_MINB) tt_brick_kernel(TTParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TTSmem& s = *reinterpret_cast<TTSmem*>(smem_raw);
    float* tile = reinterpret_cast<float*>(smem_raw + sizeof(TTSmem));
    const Scene& sc = p.sc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nbi = (sc.n1 + BI - 1) / BI, nbj = (sc.n2 + BJ - 1) / BJ;
    int b = blockIdx.x;
    const int bi = b % nbi;
    b /= nbi;
    const int bj = b % nbj, bk = b / nbj;
    const int i0 = bi * BI, j0 = bj * BJ, k0 = bk * BK;
    const int i1 = min(i0 + BI, sc.n1), j1 = min(j0 + BJ, sc.n2), k1 = min(k0 + BK, sc.n3);
    const int vg0 = p.view_begin + blockIdx.y * p.views_per_group;
    const int vg1 = min(vg0 + p.views_per_group, p.view_begin + p.view_count);
    if (vg0 >= vg1) return;
    const size_t plane = size_t(sc.n1) * sc.n2;
    if (tid == 0) {
        s.mu_abs_max = 0.f;
        s.nonfinite = 0;
    }
    __syncthreads();
    float abs_max = 0.f;
    for (int idx = tid; idx < NCOL * BK; idx += NT) {
        const int kk = idx / NCOL, c = idx % NCOL;
        const int i = i0 + (c % BI), j = j0 + (c / BI), k = k0 + kk;
        float val = 0.f;
        if (FWD && i < i1 && j < j1 && k < k1)
            val = __ldg(p.vol_in + size_t(k) * plane + size_t(j) * sc.n1 + i);
        s.vox[c * MUS + kk] = val;
        if (!isfinite(val)) s.nonfinite = 1;
        abs_max = fmaxf(abs_max, fabsf(val));
    }
    if (FWD) {
        for (int o = 16; o > 0; o >>= 1) abs_max = fmaxf(abs_max, __shfl_xor_sync(0xffffffffu, abs_max, o));
        if (lane == 0) atomicMax(reinterpret_cast<int*>(&s.mu_abs_max), __float_as_int(abs_max));
    }
    int* itile = reinterpret_cast<int*>(tile);  // forward: fixed-point accumulators
    const int rows = sc.rows, cols = sc.cols;
    const size_t npx = size_t(rows) * cols;
    for (int v = vg0; v < vg1; ++v) {
        const ViewConst& vc = p.views[v];
        const size_t vloc = size_t(v - p.view_begin);
        __syncthreads();
        if (tid < NCOL) {
            const int c = tid, i = i0 + (c % BI), j = j0 + (c / BI);
            int cnt = 0, nf = 0;
            if (i < i1 && j < j1) {
                float f1[MAXN];
                double Q0;
                float4 axc;
                float2 amp;
                cnt = column_footprint(vc, sc, i, j, f1, nf, Q0, axc, amp, p.amplitude);
                for (int q = 0; q < MAXN; ++q) s.f1[q * NCOL + c] = q < cnt ? f1[q] : 0.f;
                s.Q0[c] = Q0;
                // chi2 anchor of the column's first layer, split so the
                // voxel loop runs in float32 (cvp_device.cuh column_anchor)
                const ColumnAnchor an = column_anchor<true>(vc.pp2, sc.minz + (k0 + 0.5) * sc.a3 - vc.s3,
                                                            Q0, sc.a3);
                s.anchor[c] = make_int4(an.M0, __float_as_int(an.f0), __float_as_int(an.dh),
                                        __float_as_int(an.dl));
                s.ax[c] = axc;
                s.amp[c] = amp;
            }
            s.n0[c] = nf;
            s.nn[c] = cnt;
        } else {
            if (tid >= NT - BK) {
                // per-layer dz of this view (float64 -> float32 once per layer)
                const int kk = tid - (NT - BK);
                s.dz[kk] = float(sc.minz + (k0 + kk + 0.5) * sc.a3 - vc.s3);
            }
            if (tid == NCOL) {
                // footprint rectangle of the brick (corner projections)
                double cmin = INFINITY, cmax = -INFINITY, rmin = INFINITY, rmax = -INFINITY;
                double dn = INFINITY, df = -INFINITY, zmax = 0.0;
                bool fixed_ok = true;
                for (int q = 0; q < 8; ++q) {
                    const double x = sc.minx + ((q & 1) ? i1 : i0) * sc.a1 - vc.sx;
                    const double y = sc.miny + ((q & 2) ? j1 : j0) * sc.a2 - vc.sy;
                    const double z = sc.minz + ((q & 4) ? k1 : k0) * sc.a3 - vc.s3;
                    const double d = vc.w3x * x + vc.w3y * y;
                    const double c1 = (vc.w1x * x + vc.w1y * y) / d, c2 = vc.pp2 - z * vc.f_over_b2 / d;
                    cmin = fmin(cmin, c1);
                    cmax = fmax(cmax, c1);
                    rmin = fmin(rmin, c2);
                    rmax = fmax(rmax, c2);
                    dn = fmin(dn, d);
                    df = fmax(df, d);
                    zmax = fmax(zmax, fabs(z));
                }
                if (FWD) {
                    // Fixed-point scale: bound on any pixel's partial sum from
                    // this brick, sum_j mu_j a_j F1_j(n) F2_j(m):
                    //   a_j <= diag_xy * sqrt(1 + (v_max b2 / f)^2) (A1/A2 amplitude);
                    //   sum over columns of F1(n) <= BI + BJ (a ray crosses at most
                    //     BI + BJ cells of the brick's base grid; unit-height trapezoids);
                    //   sum over layers of F2(m) <= W/delta + 1 (trapezoid support
                    //     over the layer spacing, both in rows).
                    const double diag = sqrt(sc.a1 * sc.a1 + sc.a2 * sc.a2);
                    const double vmax = fmax(vc.pp2, double(rows - 1) - vc.pp2) + 1.0;
                    const double amax = diag * sqrt(1.0 + vmax * vmax * vc.b2 * vc.b2 / (vc.f * vc.f));
                    const double wd = (df / dn) * (1.0 + 2.0 * zmax * (df - dn) / (df * sc.a3));
                    const double bound = double(s.mu_abs_max) * amax * double(BI + BJ) * (wd + 2.0) * 1.05;
                    const double q = (bound > 0.0 && dn > 0.0) ? 1073741824.0 / bound : 0.0;
                    // NaN / Inf voxels or a scale outside the normal float32
                    // range: this (brick, view) scatters with float atomics
                    fixed_ok = (!s.nonfinite && q > 0.0 && q < 3.0e38 && float(q) >= 1.17549435e-38f) ||
                               (s.mu_abs_max == 0.f && !s.nonfinite);
                    s.qscale = fixed_ok && q > 0.0 ? float(q) : 0.f;
                }
                const int n0 = max(int(ceil(cmin - 0.5)) - 1, 0), n1 = min(int(floor(cmax + 0.5)) + 1, cols - 1);
                const int m0 = max(int(ceil(rmin - 0.5)) - 1, 0), m1 = min(int(floor(rmax + 0.5)) + 1, rows - 1);
                const int tr = max(m1 - m0 + 1, 0), tc = max(n1 - n0 + 1, 0);
                s.tile_m0 = m0;
                s.tile_n0 = n0;
                s.tile_rows = tr;
                s.tile_cols = tc;
                s.tile_stride = tr | 1;
                s.tile_ok = (tr > 0 && tc > 0 && (tr | 1) * tc <= p.tile_cap && fixed_ok) ? 1 : 0;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(NT - NCOL) : "memory");
            if (s.tile_ok) {
                const int tm0 = s.tile_m0, tn0 = s.tile_n0, trows = s.tile_rows, tcols = s.tile_cols;
                const int tstride = s.tile_stride;
                if (FWD) {
                    for (int idx = tid - NCOL; idx < tstride * tcols; idx += NT - NCOL) itile[idx] = 0;
                } else {
                    const float* img = p.proj_in + vloc * npx;
                    for (int idx = tid - NCOL; idx < trows * tcols; idx += NT - NCOL) {
                        const int r = idx / tcols, cc = idx % tcols;
                        tile[cc * tstride + r] = __ldg(img + size_t(tm0 + r) * cols + (tn0 + cc));
                    }
                }
            }
        }
        __syncthreads();
        const int tm0 = s.tile_m0, tn0 = s.tile_n0, trows = s.tile_rows, tcols = s.tile_cols;
        const int tstride = s.tile_stride;
        const bool tile_ok = s.tile_ok != 0;
        if (trows == 0 || tcols == 0) continue;  // the brick misses the detector in this view
        const float b2 = float(vc.b2);
        float* out_img = FWD ? p.proj_out + vloc * npx : nullptr;
        const float* in_img = FWD ? nullptr : p.proj_in + vloc * npx;
        for (int cq = warp; cq < NCOL * NH; cq += NWARP) {
            const int c = cq / NH, hf = cq % NH;
            const int cnt = s.nn[c];
            if (cnt == 0) continue;
            const int kk = lane + 32 * hf;
            const int k = k0 + kk;
            const bool kvalid = k < k1;
            const float mu = FWD ? s.vox[c * MUS + kk] : 0.f;
            if (FWD && !__any_sync(0xffffffffu, kvalid && mu != 0.f)) continue;
            const float dz = s.dz[kk];
            // anchor chi2(zc) at the base-centre depth: integer row m_ref and
            // float32 remainders u = chi2 - m_ref, pm = pp2 - m_ref
            int m_ref;
            float u, pm;
            if (FWD) {
                // float64 per voxel (the float32 split below measured 3% slower
                // here: its extra live state spills in the forward)
                const double c0 = fma(-(sc.minz + (k + 0.5) * sc.a3 - vc.s3), s.Q0[c], vc.pp2);
                const double mr = rint(c0);
                m_ref = int(mr);
                u = float(c0 - mr);
                pm = float(vc.pp2 - mr);
            } else {
                // the column's float64 split, float32 per voxel (exact to
                // ~1e-7 px; cvp_device.cuh anchor_at): backward +6%
                const int4 a4 = s.anchor[c];
                const ColumnAnchor an{a4.x, __int_as_float(a4.y), __int_as_float(a4.z), __int_as_float(a4.w)};
                float Mf_unused;
                anchor_at(an, float(vc.pp2), float(kk), m_ref, Mf_unused, u, pm);
            }
            const float4 axc = s.ax[c];
            float t0 = u + dz * axc.x - axc.z, t1 = u + dz * axc.x + axc.z;
            float t2 = u + dz * axc.y - axc.w, t3 = u + dz * axc.y + axc.w;
            sort4(t0, t1, t2, t3);
            int mf = m_ref + int(ceilf(t0 - 0.5f)), ml = m_ref + int(floorf(t3 + 0.5f));
            mf = max(mf, 0);
            ml = min(ml, rows - 1);
            const float2 amp = s.amp[c];
            const int nfirst = s.n0[c];
            const int ncache = min(cnt, MAXN);
            // ramp reciprocals once per voxel (trap_cdf semantics: zero-width ramps)
            const float w1 = t1 - t0, w3 = t3 - t2;
            const float r1 = w1 > 0.f ? 0.5f * frcp(w1) : 0.f, r3 = w3 > 0.f ? 0.5f * frcp(w3) : 0.f;
            auto cdf = [&](float x) {
                const float c1 = fminf(fmaxf(x, t0), t1);
                const float mid = fminf(fmaxf(x, t1), t2) - t1;
                const float c3 = fminf(fmaxf(x, t2), t3);
                return (c1 - t0) * (c1 - t0) * r1 + mid + (c3 - t2) * (w3 + t3 - c3) * r3;
            };
            const float ampA1 = AMP2 ? 0.f : amp.x * sqrtf(1.f + (u - pm) * (u - pm) * b2 * b2 * amp.y);
            float acc = 0.f;
            const bool active = kvalid && (!FWD || mu != 0.f);
            const float muq = FWD ? mu * s.qscale : 0.f;  // fixed-point scale folded into mu
            // the whole (rows x columns) footprint of this voxel inside the tile?
            const bool inside = tile_ok && mf >= tm0 && ml < tm0 + trows && nfirst >= tn0 &&
                                nfirst + ncache <= tn0 + tcols;
            if (active && cnt <= MAXN) {
                float g_prev = cdf(float(mf - m_ref) - 0.5f);
                for (int m = mf; m <= ml; ++m) {
                    const float g = cdf(float(m - m_ref) + 0.5f);
                    const float f2 = g - g_prev;
                    g_prev = g;
                    if (!(f2 > 0.f)) continue;
                    float a;
                    if (AMP2) {
                        const float vm = float(m - m_ref) - pm;  // (m - pp2)
                        a = amp.x * sqrtf(1.f + vm * vm * b2 * b2 * amp.y);
                    } else {
                        a = ampA1;
                    }
                    const float wrow = a * f2;
                    if (inside) {
                        const int off = (nfirst - tn0) * tstride + (m - tm0);
                        // unrolled: ncache is the column's (warp-uniform) width
#pragma unroll
                        for (int q = 0; q < MAXN; ++q) {
                            if (q < ncache) {
                                const float w = wrow * s.f1[q * NCOL + c];
                                if (FWD)
                                    red_s32(itile + off + q * tstride, __float2int_rn(muq * w));
                                else
                                    acc = fmaf(w, tile[off + q * tstride], acc);
                            }
                        }
                    } else {
                        for (int q = 0; q < ncache; ++q) {
                            const int n = nfirst + q;
                            const float w = wrow * s.f1[q * NCOL + c];
                            const int r = m - tm0, cc = n - tn0;
                            const bool in_tile = tile_ok && unsigned(r) < unsigned(trows) &&
                                                 unsigned(cc) < unsigned(tcols);
                            if (FWD) {
                                if (in_tile)
                                    red_s32(itile + cc * tstride + r, __float2int_rn(muq * w));
                                else
                                    atomicAdd(out_img + size_t(m) * cols + n, mu * w);
                            } else {
                                acc += w * (in_tile ? tile[cc * tstride + r]
                                                    : __ldg(in_img + size_t(m) * cols + n));
                            }
                        }
                    }
                }
            }
            if (cnt > MAXN && active) {
                // very wide transaxial footprint: walk every (n, m) pair directly
                const WideColumn wc = wide_column(vc, sc, i0 + (c % BI), j0 + (c / BI));
                float g_prev = cdf(float(mf - m_ref) - 0.5f);
                for (int m = mf; m <= ml; ++m) {
                    const float g = cdf(float(m - m_ref) + 0.5f);
                    const float f2 = g - g_prev;
                    g_prev = g;
                    if (!(f2 > 0.f)) continue;
                    const float vm = float(m - m_ref) - pm;
                    const float a = AMP2 ? amp.x * sqrtf(1.f + vm * vm * b2 * b2 * amp.y) : ampA1;
                    float h_prev = trap_cdf(float(wc.nlo) - 0.5f, wc.s0, wc.s1, wc.s2, wc.s3);
                    for (int nn = wc.nlo; nn <= wc.nhi; ++nn) {
                        const float hh = trap_cdf(float(nn) + 0.5f, wc.s0, wc.s1, wc.s2, wc.s3);
                        const float w = a * f2 * (hh - h_prev);
                        h_prev = hh;
                        const int n = wc.nr + nn;
                        if (FWD)
                            atomicAdd(out_img + size_t(m) * cols + n, mu * w);
                        else
                            acc += w * __ldg(in_img + size_t(m) * cols + n);
                    }
                }
            }
            if (!FWD && kvalid) s.vox[c * MUS + kk] += acc;
        }
        if (FWD && tile_ok) {
            __syncthreads();
            const float inv_qs = s.qscale > 0.f ? 1.f / s.qscale : 0.f;
            for (int idx = tid; idx < trows * tcols; idx += NT) {
                const int r = idx / tcols, cc = idx % tcols;
                const int q = itile[cc * tstride + r];
                if (q != 0) atomicAdd(out_img + size_t(tm0 + r) * cols + (tn0 + cc), float(q) * inv_qs);
            }
        }
    }
    if (!FWD) {
        __syncthreads();
        for (int idx = tid; idx < NCOL * BK; idx += NT) {
            const int kk = idx / NCOL, c = idx % NCOL;
            const int i = i0 + (c % BI), j = j0 + (c / BI), kq = k0 + kk;
            if (i < i1 && j < j1 && kq < k1) {
                float* dst = p.vol_out + size_t(kq) * plane + size_t(j) * sc.n1 + i;
                const float val = s.vox[c * MUS + kk];
                if (p.atomic_out)
                    atomicAdd(dst, val);
                else if (p.accumulate)
                    *dst += val;
                else
                    *dst = val;
            }
        }
    }
}

// detector tile: what is left of a quarter of the SM's 228 KB of shared
// memory (four resident CTAs); bricks whose footprint does not fit use the
// global-memory path
constexpr int kTileCap = int((228 * 1024 / TT_MINB - 1024 - sizeof(TTSmem)) / sizeof(float));

}  // namespace

cudaError_t launch_tt(const TTLaunch& L, bool forward, cudaStream_t stream) {
    if (L.view_count <= 0) {
        if (!forward && !L.accumulate)
            return cudaMemsetAsync(L.vol_out, 0,
                                   sizeof(float) * size_t(L.sc.n1) * L.sc.n2 * L.sc.n3, stream);
        return cudaSuccess;
    }
    const Scene& sc = L.sc;
    const int dyn = int(sizeof(TTSmem)) + kTileCap * int(sizeof(float));
    const int nbricks = ((sc.n1 + BI - 1) / BI) * ((sc.n2 + BJ - 1) / BJ) * ((sc.n3 + BK - 1) / BK);
    int groups = 1;
    const int target = 148 * 2 * 2;
    if (nbricks < target) groups = std::min(L.view_count, (target + nbricks - 1) / nbricks);
    const int per = (L.view_count + groups - 1) / groups;
    groups = (L.view_count + per - 1) / per;
    TTParams p;
    p.sc = sc;
    p.views = L.views;
    p.vol_in = L.vol_in;
    p.vol_out = L.vol_out;
    p.proj_in = L.proj_in;
    p.proj_out = L.proj_out;
    p.view_begin = L.view_begin;
    p.view_count = L.view_count;
    p.views_per_group = per;
    p.amplitude = L.amplitude;
    p.tile_cap = kTileCap;
    p.accumulate = L.accumulate;
    p.atomic_out = groups > 1 ? 1 : 0;
    cudaError_t e;
    dim3 grid(nbricks, groups);
    if (forward) {
        e = cudaMemsetAsync(L.proj_out, 0, sizeof(float) * size_t(sc.rows) * sc.cols * L.view_count,
                            stream);
        if (e != cudaSuccess) return e;
        auto kern = L.amplitude ? tt_brick_kernel<true, true> : tt_brick_kernel<true, false>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        if (e != cudaSuccess) return e;
        kern<<<grid, NT, dyn, stream>>>(p);
    } else {
        if (groups > 1 && !L.accumulate) {
            e = cudaMemsetAsync(L.vol_out, 0, sizeof(float) * size_t(sc.n1) * sc.n2 * sc.n3, stream);
            if (e != cudaSuccess) return e;
        }
        auto kern = L.amplitude ? tt_brick_kernel<false, true> : tt_brick_kernel<false, false>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        if (e != cudaSuccess) return e;
        kern<<<grid, NT, dyn, stream>>>(p);
    }
    return cudaGetLastError();
}

}  // namespace cvpb
