// CVP forward (scatter) and backward (gather) kernels for sm_100a.
//
// Reference: /root/reference/proj/src/cvp.cpp forward_view (:357-412),
// backward_view (:414-458), project/backproject_cvp_impl (:460-500).
//
// Work decomposition:
//   cut table  cut_table_kernel computes the column cuts of every voxel column
//              once per view (float64 world quantities in exact mode);
//   bricks     one CTA owns BI x BJ voxel columns x BK voxels along x3
//              (8 x 16 x 64, bricks numbered k-fastest) and loops over views:
//   G-phase    one thread per column loads its cuts from the table into
//              shared memory and splits its chi2 anchor; the other warps bound
//              the brick's detector footprint and (backward) stage the tile;
//   V-phase    warp w walks columns w, w+8, ...; each lane carries the voxels
//              k = lane and lane + 32 through every cut, and each
//              (voxel, cut, row) record is
//                forward:  added (int32 fixed point) into a shared-memory
//                          detector tile (column-major, odd stride),
//                backward: gathered from a shared-memory copy of the scaled
//                          image footprint (no atomics);
//   flush      forward: the tile is added to HBM with one float atomic per
//              touched pixel and re-zeroed; the phase-2 pixel scale
//              (cvp.cpp:473-474) is one streaming pass after the launch.
// The brick's attenuation values (forward) / accumulators (backward) stay in
// shared memory across all views, so HBM sees the volume once per launch.
//
// Build parameters (defaults are the measured optimum on B200, see
// profiles/ncu_r01.md): CVP_BI / CVP_BJ / CVP_BK brick shape, CVP_NV voxels
// per lane per cut pass, CVP_NT threads, CVP_MINB resident CTAs per SM,
// CVP_MAXC (kernels.hpp) cut slots per column.
#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "cvp_device.cuh"
#include "kernels.hpp"

// The file is compiled three times (Makefile): the default brick shape
// (8x16x64, 256 threads, three CTAs per SM), shape B (CVP_CFG_B: 8x8x64 at
// four CTAs per SM) and shape C (CVP_CFG_C: 8x24x64, 384 threads, two CTAs
// per SM); the brick-dependent entry points of the extra copies carry a _b /
// _c suffix and the shape-independent ones exist once.
#if defined(CVP_CFG_B)
#define CVP_PUB(name) name##_b
#elif defined(CVP_CFG_C)
#define CVP_PUB(name) name##_c
#else
#define CVP_PUB(name) name
#endif

namespace cvpb {

namespace {

#ifndef CVP_BJ
#define CVP_BJ 16
#endif
#ifndef CVP_BK
#define CVP_BK 64
#endif
#ifndef CVP_BI
#define CVP_BI 8
#endif
constexpr int BI = CVP_BI, BJ = CVP_BJ, BK = CVP_BK;
constexpr int NCOL = BI * BJ;           // voxel columns per brick
#ifndef CVP_NT
#define CVP_NT 256
#endif
constexpr int NT = CVP_NT;              // threads per CTA
constexpr int NWARP = NT / 32;
constexpr int NH = BK / 32;             // voxels per lane along x3 (lane, lane + 32, ...)
static_assert(BK % 32 == 0 && BK <= 128, "anchor split is exact for kk < 128");
static_assert(NCOL <= NT, "one G-phase thread per column");
static_assert(NT - BK >= NCOL, "per-layer dz threads lie outside the G-phase");
#ifndef CVP_MINB
#define CVP_MINB 3                      // resident CTAs per SM (80 registers)
#endif
#ifndef CVP_NV
#define CVP_NV 2
#endif
constexpr int NV = CVP_NV;              // voxels per lane per cut pass (kk = lane + 32 t)
static_assert(NH % NV == 0, "whole voxel groups per column");

// Per-lane state of one voxel in the V-phase.
struct VoxState {
    int Mi;
    float u0h, pmh, dz, dz2e28, mu, muq, inv_r2_fixed, acc;  // (row as float: float(Mi), exact)
    uint32_t vaddr;
    bool kvalid, active;
};
constexpr int MAXC = kCutSlots;         // cuts cached per column; more are recomputed
constexpr int MUS = BK + 1;             // padded column stride of the voxel tile

// Column cuts of every voxel column under views [v0, v0 + nv), computed once
// per (view, column) by cut_table_kernel instead of once per brick: the
// G-phase of a brick becomes a load. Index (v - v0) * ncols + j * n1 + i;
// cut slot q of a column at ((v - v0) * MAXC + q) * ncols + column.
struct CutTable {
    int* count;
    double* Q0;
    float* rho2c;
    float4* cutA;  // {A, g, rho2, shw}
    float4* cutB;  // {kc, tr_a, tr_b, n (bits)}
    int v0, nv;
    int ncols;
};

struct CvpParams {
    Scene sc;
    CutTable t;
    const ViewConst* views;
    const float* scales;      // [slots][rows*cols]
    const float* vol_in;      // forward input
    float* vol_out;           // backward output
    const double* vol_in64;   // forward input, mapped host float64 (instead of vol_in)
    float* vol_copy;          // with vol_in64: float32 copy of the input left here
    double* vol_out64;        // backward output, mapped host float64 (instead of vol_out)
    const float* proj_in;     // backward input (view_begin-relative)
    float* proj_out;          // forward output (view_begin-relative)
    int view_begin, view_count, views_per_group;
    int corr, per_row_r;
    float h;                  // a3 / 2
    int tile_cap;
    int accumulate;           // backward: add into vol_out
    int atomic_out;           // backward: several view groups -> atomicAdd
    // forward, ExecPolicy::deterministic: bricks merge into an int64
    // fixed-point stack (view_begin-relative) at the launch-wide scale *det_g
    // (integer adds commute: the result is bit-reproducible); *det_g == 0
    // (non-finite volume) falls back to the float atomics
    unsigned long long* det_acc;
    const double* det_g;
    SlabTargets tg;           // backward fused with a reduce-scatter (tg.n > 0)
    int* err;
};

// Shared-memory layout (dynamic). Cut records are two float4 each so a warp
// reads one record with two broadcast LDS.128.
struct Smem {
    float4 cutA[MAXC * NCOL];  // {A, g, rho2, shw}
    float4 cutB[MAXC * NCOL];  // {kc, tr_a, tr_b, n (bits)}
    int4 anchor[NCOL];        // ColumnAnchor {M0, f0, dh, dl} of each column
    float rho2c[NCOL];
    float dz[BK];             // zc - s3 of the brick's voxel layers under this view
    int count[NCOL];          // cuts per column under the current view
    int nonzero[NCOL];        // forward: the column holds a nonzero attenuation
    float vox[NCOL * MUS];    // forward: mu; backward: accumulators
    float* img;               // this view's image (forward: output, backward: input)
    unsigned long long* dimg; // forward, deterministic: this view's int64 image (else null)
    double det_g;             // forward, deterministic: fixed-point scale (0: float atomics)
    const float* scale;       // backward: this view's phase-2 factors
    int tile_m0, tile_n0, tile_rows, tile_cols, tile_stride, tile_ok;
    float mu_abs_max;         // forward: max |mu| over the brick
    int nonfinite;            // forward: the brick holds a NaN / Inf attenuation
    float qscale;             // forward: fixed-point scale of this (brick, view)
    int walk_mode;            // 0: general row walk; 1 / 2 / 3: walk_rows_fast<1 / 2 / 3>;
                              // 5 / 6 / 7: the same with rows off the detector dropped
};

// 32-bit shared-window addressing for the hot paths: with 80 registers the
// compiler otherwise rematerialises the generic->shared window base
// (S2R SR_CgaCtaId + LEA) at every access.
__device__ __forceinline__ uint32_t saddr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void red_s32(uint32_t a, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// red.shared.add only where pred != 0 and v != 0 (no branch around it)
__device__ __forceinline__ void red_s32_if(uint32_t a, int v, int pred) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.s32 p, %2, 0;\n\t"
        "setp.ne.and.s32 q, %1, 0, p;\n\t"
        "@q red.shared.add.s32 [%0], %1;\n\t}" ::"r"(a), "r"(v), "r"(pred) : "memory");
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ CutRec load_cut(uint32_t sbase, int slot) {
    const float4 a = lds_f32x4(sbase + uint32_t(offsetof(Smem, cutA)) + 16u * slot);
    const float4 b = lds_f32x4(sbase + uint32_t(offsetof(Smem, cutB)) + 16u * slot);
    CutRec r;
    r.A = a.x;
    r.g = a.y;
    r.rho2 = a.z;
    r.shw = a.w;
    r.kc = b.x;
    r.tr_a = b.y;
    r.tr_b = b.z;
    r.n = __float_as_int(b.w);
    return r;
}

// Division on the footprint thread's critical path: the approximate device
// form (~2 ulp; the footprint needs pixel accuracy, its rigorous bounds
// carry >= 1e-4 relative slack).
__host__ __device__ __forceinline__ float fdiv_fp(float a, float b) {
#ifdef __CUDA_ARCH__
    return __fdividef(a, b);
#else
    return a / b;
#endif
}

// Detector rectangle that contains every record a voxel of the brick can
// emit under view vc: chi1 over the brick's base corners; chi2 over its z
// range and its depth range widened by half a voxel-base diagonal (bound on
// the elevation rectangle's depth spread |hw|*halfw). One extra column and
// two extra rows of margin absorb rounding (the evaluation is float32: the
// rectangle only needs pixel accuracy, and the same function sizes the tile
// in tile_need_kernel); anything outside still lands correctly through the
// global fallback path. The returned depths are the brick base's corner
// depth range (unwidened).
__host__ __device__ inline void brick_footprint(const ViewConst& vc, const Scene& sc, int i0, int i1,
                                                int j0, int j1, int k0, int k1, int& m0, int& m1,
                                                int& n0, int& n1, float* depth_min = nullptr,
                                                float* depth_max = nullptr,
                                                bool* rows_inside = nullptr, int* r0_out = nullptr,
                                                int* r1_out = nullptr, float margin_in = -1.f) {
    // corner offsets from the source in float32 (|offset| <~ 1e3 mm: ~6e-5 mm)
    const float xs[2] = {float(sc.minx + i0 * sc.a1 - vc.sx), float(sc.minx + i1 * sc.a1 - vc.sx)};
    const float ys[2] = {float(sc.miny + j0 * sc.a2 - vc.sy), float(sc.miny + j1 * sc.a2 - vc.sy)};
    const float w1x = float(vc.w1x), w1y = float(vc.w1y), w3x = float(vc.w3x), w3y = float(vc.w3y);
    float cmin = INFINITY, cmax = -INFINITY, dmin = INFINITY, dmax = -INFINITY;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            const float d = w3x * xs[a] + w3y * ys[b];
            const float c1 = fdiv_fp(w1x * xs[a] + w1y * ys[b], d);
            cmin = fminf(cmin, c1);
            cmax = fmaxf(cmax, c1);
            dmin = fminf(dmin, d);
            dmax = fmaxf(dmax, d);
        }
    if (depth_min) *depth_min = dmin;
    if (depth_max) *depth_max = dmax;
    if (rows_inside) *rows_inside = false;
    // (half the voxel-base diagonal; the kernel passes it precomputed)
    const float margin = margin_in >= 0.f ? margin_in : float(0.5 * sqrt(sc.a1 * sc.a1 + sc.a2 * sc.a2));
    const float dlo = dmin - margin, dhi = dmax + margin;
    if (!(dlo > 0.f) || !(cmin > -1e7f) || !(cmax < 1e7f)) {
        m0 = 1;
        m1 = 0;
        n0 = 1;
        n1 = 0;
        return;
    }
    const float fb2 = float(vc.f_over_b2), pp2 = float(vc.pp2);
    const float z0 = float(sc.minz + k0 * sc.a3 - vc.s3), z1 = float(sc.minz + k1 * sc.a3 - vc.s3);
    const float rlo = fdiv_fp(1.f, dlo), rhi = fdiv_fp(1.f, dhi);
    // chi2 = pp2 - z fb2 / d is monotone in z and in 1/d: extremes at the corners
    float rmin = INFINITY, rmax = -INFINITY;
    for (float z : {z0, z1})
        for (float r : {rlo, rhi}) {
            const float c2 = pp2 - z * fb2 * r;
            rmin = fminf(rmin, c2);
            rmax = fmaxf(rmax, c2);
        }
    if (!(rmin > -1e7f) || !(rmax < 1e7f)) {
        m0 = 1;
        m1 = 0;
        n0 = 1;
        n1 = 0;
        return;
    }
    n0 = max(int(ceilf(cmin - 0.5f)) - 1, 0);
    n1 = min(int(floorf(cmax + 0.5f)) + 1, sc.cols - 1);
    // two rows of margin: the fast row walk (walk_rows_fast) emits up to one
    // row past a voxel's range, whose own bound carries float slack
    const int r0 = int(ceilf(rmin - 0.5f)) - 2, r1 = int(floorf(rmax + 0.5f)) + 2;
    m0 = max(r0, 0);
    m1 = min(r1, sc.rows - 1);
    if (rows_inside) *rows_inside = r0 >= 0 && r1 <= sc.rows - 1;
    if (r0_out) *r0_out = r0;  // the row range before clamping to the detector
    if (r1_out) *r1_out = r1;
}

// Cuts q0 .. q0 + kOverflowCap - 1 of column (i, j) under view *vc — those
// past the MAXC that the cut table caches — recomputed out of line. Inlined,
// the float64 column geometry (column_cuts) set the register allocation of
// the whole V-phase and forced 100-150 B of spills into every kernel variant
// (reloaded on the hot cut loop); behind a call the rare path pays for its
// own registers at the call site only.
constexpr int kOverflowCap = 8;
template <bool EXACT>
__device__ __noinline__ void overflow_cuts(const ViewConst* vc, Scene sc, int i, int j, int corr,
                                           int q0, CutRec* out) {
    ColumnRec col;
    int idx = 0;
    column_cuts<EXACT>(*vc, sc, i, j, true, corr != 0, col, [&](const CutRec& r) {
        if (idx >= q0 && idx < q0 + kOverflowCap) out[idx - q0] = r;
        ++idx;
    });
}

// One voxel-cut whose column is off the brick's detector tile (tile overflow
// or a column outside the footprint): records go straight to HBM — float
// atomics, or the int64 merge stack in deterministic mode — and the backward
// gathers the scaled image from L2. Out of line for the same reason as
// overflow_cuts. Returns the backward's sum of image * weight.
template <bool FWD, int NR>
__device__ __noinline__ float offtile_walk(CutRec r, int Mi, float Mf, float uh, float pmh, float dz,
                                           float h, float sh, int per_row_r, float inv_r2_fixed,
                                           int rows, int cols, float mu, float* img,
                                           const float* scl, unsigned long long* dimg, double g) {
    float cut_acc = 0.f;
    auto emit = [&](int m, float wr) {
        // the walk's padding emit may sit one row past the detector
        const size_t px = size_t(min(m, rows - 1)) * cols + r.n;
        if (FWD) {
            // zero records (padding row, empty range, mu = 0) skip the atomic
            if (wr != 0.f && mu != 0.f) {
                const float val = mu * r.A * wr;
                if (dimg)
                    atomicAdd(dimg + px, static_cast<unsigned long long>(__double2ll_rn(double(val) * g)));
                else
                    atomicAdd(img + px, val);
            }
        } else {
            cut_acc = fmaf(__ldg(img + px) * __ldg(scl + px), wr, cut_acc);
        }
    };
    walk_rows<true, decltype(emit)&, true, NR>(r, Mi, Mf, uh, pmh, dz, h, sh, per_row_r != 0,
                                               inv_r2_fixed, rows, emit);
    return cut_acc;
}

// CORR: elevation correction option; CCR: radius estimate (cvp.hpp:17-22):
// 0 VoxelCenter, 1 CutCentroid per row segment, 2 CutCentroid in relaxed
// precision (per voxel-cut where the brick allows it) — compile-time so the
// unused paths cost no registers.
template <bool EXACT, bool FWD, bool CORR, int CCR, int NR>
__global__ void __launch_bounds__(NT, CVP_MINB) cvp_brick_kernel(CvpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    float* tile = reinterpret_cast<float*>(smem_raw + sizeof(Smem));
    int* itile = reinterpret_cast<int*>(tile);  // forward: fixed-point accumulators
    // opaque to the compiler, so it stays in a register instead of being
    // re-derived from SR_CgaCtaId in every cut
    uint32_t sbase;
    asm volatile("mov.u32 %0, %1;" : "=r"(sbase) : "r"(saddr(smem_raw)));
    const uint32_t tbase = sbase + uint32_t(sizeof(Smem));  // detector tile

    const Scene& sc = p.sc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nbi = (sc.n1 + BI - 1) / BI, nbj = (sc.n2 + BJ - 1) / BJ;
    // k fastest: the bricks of one column stack run together and share the
    // cut-table reads in L2
    const int nbk = (sc.n3 + BK - 1) / BK;
    int b = blockIdx.x;
    const int bk = b % nbk;
    b /= nbk;
    const int bi = b % nbi;
    const int bj = b / nbi;
    const int i0 = bi * BI, j0 = bj * BJ, k0 = bk * BK;
    const int i1 = min(i0 + BI, sc.n1), j1 = min(j0 + BJ, sc.n2), k1 = min(k0 + BK, sc.n3);

    const int vg0 = p.view_begin + blockIdx.y * p.views_per_group;
    const int vg1 = min(vg0 + p.views_per_group, p.view_begin + p.view_count);
    if (vg0 >= vg1) return;

    const size_t plane = size_t(sc.n1) * sc.n2;
    // Stage the brick's voxels: [column][k] with odd stride (bank-conflict free).
    if (tid < NCOL) s.nonzero[tid] = 0;
    if (tid == 0) {
        s.mu_abs_max = 0.f;
        s.nonfinite = 0;
        s.det_g = (FWD && p.det_g) ? *p.det_g : 0.0;
    }
    // forward: the fixed-point tile starts zeroed and every flush re-zeroes
    // the pixels it reads, so views need no zeroing pass of their own
    if (FWD)
        for (int idx = tid; idx < p.tile_cap; idx += NT) itile[idx] = 0;
    __syncthreads();
    float abs_max = 0.f;
    for (int idx = tid; idx < NCOL * BK; idx += NT) {
        const int kk = idx / NCOL, c = idx % NCOL;
        const int i = i0 + (c % BI), j = j0 + (c / BI), k = k0 + kk;
        float val = 0.f;
        if (FWD && i < i1 && j < j1 && k < k1) {
            const size_t off = size_t(k) * plane + size_t(j) * sc.n1 + i;
            if (p.vol_in64) {
                val = float(p.vol_in64[off]);
                if (p.vol_copy) p.vol_copy[off] = val;
            } else {
                val = __ldg(p.vol_in + off);
            }
            if (val != 0.f) s.nonzero[c] = 1;
            if (!isfinite(val)) s.nonfinite = 1;
            abs_max = fmaxf(abs_max, fabsf(val));
        }
        s.vox[c * MUS + kk] = val;
    }
    if (FWD) {
        for (int o = 16; o > 0; o >>= 1) abs_max = fmaxf(abs_max, __shfl_xor_sync(0xffffffffu, abs_max, o));
        // non-negative floats order like their bit patterns
        if (lane == 0) atomicMax(reinterpret_cast<int*>(&s.mu_abs_max), __float_as_int(abs_max));
    }

    const int rows = sc.rows, cols = sc.cols;
    const size_t npx = size_t(rows) * cols;
    const float h = p.h;
    // forward: per-scene constants of the footprint thread once per CTA (no
    // float64 square root / divisions on the per-view G-phase critical path:
    // P +2% at c3); the backward recomputes them per view (held across the
    // view loop they cost it 2-8% in register pressure)
    const float diag_pre = FWD ? float(sqrt(sc.a1 * sc.a1 + sc.a2 * sc.a2)) : 0.f;
    const float b1_over_b2 = FWD ? float(sc.pw / sc.ph) : 0.f;
    const double inv_a3_pre = FWD ? 1.0 / sc.a3 : 0.0;
    constexpr bool corr = CORR, per_row_r = CCR != 0;

    for (int v = vg0; v < vg1; ++v) {
        const ViewConst& vc = p.views[v];
        __syncthreads();  // previous view's V-phase / flush is complete
        // ---- backward tile prologue: stage the scaled image footprint
        // (threads t0, t0 + step, ...) ----------------------------------------
        auto tile_prologue = [&](int t0, int step) {
            if (!s.tile_ok || s.tile_rows == 0 || s.tile_cols == 0) return;
            const int tm0 = s.tile_m0, tn0 = s.tile_n0, trows = s.tile_rows, tcols = s.tile_cols;
            const int tstride = s.tile_stride;
            const float* img = s.img;
            const float* scale = s.scale;
#ifndef CVP_OLD_PROLOGUE
            // warps over tile rows, lanes over tile columns (coalesced image
            // reads, conflict-free column-major stores at the odd stride);
            // four rows in flight per thread, no integer division
            const int w0 = t0 >> 5, nw = step >> 5, ln = t0 & 31;
            // (virtual rows — tm0 < 0 or past the detector — stage zeros)
            for (int c0 = ln; c0 < tcols; c0 += 32) {
                const float* irow = img + ptrdiff_t(tm0) * cols + (tn0 + c0);
                const float* srow = scale + ptrdiff_t(tm0) * cols + (tn0 + c0);
                float* tcol = tile + c0 * tstride;
                int r = w0;
                for (; r + 3 * nw < trows; r += 4 * nw) {
                    float a[4], b[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int rr = r + u * nw;
                        const bool in = unsigned(tm0 + rr) < unsigned(rows);
                        const ptrdiff_t o = ptrdiff_t(rr) * cols;
                        a[u] = in ? __ldg(irow + o) : 0.f;
                        b[u] = in ? __ldg(srow + o) : 0.f;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) tcol[r + u * nw] = a[u] * b[u];
                }
                for (; r < trows; r += nw) {
                    const ptrdiff_t o = ptrdiff_t(r) * cols;
                    tcol[r] = unsigned(tm0 + r) < unsigned(rows) ? __ldg(irow + o) * __ldg(srow + o) : 0.f;
                }
            }
#else
            for (int idx = t0; idx < trows * tcols; idx += step) {
                const int r = idx / tcols, cc = idx % tcols;
                const size_t px = size_t(tm0 + r) * cols + (tn0 + cc);
                tile[cc * tstride + r] = __ldg(img + px) * __ldg(scale + px);
            }
#endif
        };
        // ---- G-phase: column cuts --------------------------------------
        // Warps past the G-phase columns (NCOL < NT) compute the brick
        // footprint and stage the detector tile meanwhile.
        // (backward only: the forward has no prologue — its tile is kept
        // zeroed by the flush — and moving its footprint work here spills)
        constexpr bool SPLIT = NCOL < NT && !FWD;
        auto footprint = [&]() {
            int m0, m1, n0, n1, r0u = 0, r1u = -1;
            bool fixed_ok = true, rows_inside = false;
            float dmin = 0.f, dmax = 0.f;
            const float diag = FWD ? diag_pre : float(sqrt(sc.a1 * sc.a1 + sc.a2 * sc.a2));
            brick_footprint(vc, sc, i0, i1, j0, j1, k0, k1, m0, m1, n0, n1, &dmin, &dmax, &rows_inside,
                            &r0u, &r1u, 0.5f * diag);
            const float fb2 = float(vc.f_over_b2);
            // Row-walk mode of this (brick, view): the fast walk needs every
            // voxel's rows inside the detector (no clamping), a full brick
            // along x3 (no virtual layers) and 2 tr < NB (<= NB + 1 rows) for every
            // voxel-cut, with the rigorous bound
            //   tr <= h f/(b2 (dmin - dd)) + |dz|max f dd / (b2 dmin (dmin - dd)) + 1e-5,
            // dd = diag/2 >= |hw| halfw (walk_rows_fast, cvp_device.cuh);
            // and (elevation correction) the gate dz^2 > 1e-28 rho^2
            // (cvp.cpp:353-355) true for every voxel-cut: |dz| at the layer
            // nearest the source plane against rho <= the largest source
            // distance of the brick's base corners.
            {
                int mode = 0;
                const float ddm = 0.5f * diag;
                const float dl = dmin - ddm;
                const float zlo = float(sc.minz + (k0 + 0.5) * sc.a3 - vc.s3);
                const float zhi = float(sc.minz + (k1 - 0.5) * sc.a3 - vc.s3);
                float dz_near;
                if (zlo > 0.f || zhi < 0.f) {
                    dz_near = fminf(fabsf(zlo), fabsf(zhi));
                } else {
                    // (nearest layer to the source plane: a reciprocal
                    // multiply can only pick a neighbour at a .5 tie, where
                    // both are half a layer away)
                    const double zc0 = sc.minz + (k0 + 0.5) * sc.a3 - vc.s3;
                    const double t = rint(FWD ? -zc0 * inv_a3_pre : -zc0 / sc.a3);
                    dz_near = float(fabs(sc.minz + (k0 + 0.5 + t) * sc.a3 - vc.s3));
                }
                float rho2max = 0.f;
                for (int q = 0; q < 4; ++q) {
                    const float x = float(sc.minx + ((q & 1) ? i1 : i0) * sc.a1 - vc.sx);
                    const float y = float(sc.miny + ((q & 2) ? j1 : j0) * sc.a2 - vc.sy);
                    rho2max = fmaxf(rho2max, x * x + y * y);
                }
                const bool gate_ok = !corr || dz_near * dz_near > 4e-28f * rho2max;
                if (k1 == k0 + BK && dl > 0.f && gate_ok) {
                    const float dzm = fmaxf(fabsf(zlo), fabsf(zhi));
                    const float rdl = fdiv_fp(1.f, dl);
                    const float tr = (0.5f * float(sc.a3) + fdiv_fp(dzm * ddm, dmin)) * fb2 * rdl * 1.0001f + 2e-5f;
                    mode = 2.f * tr < 0.999f ? 1 : 2.f * tr < 1.999f ? 2 : 2.f * tr < 2.999f ? 3 : 0;
                    // a brick whose rows reach past the detector's top or
                    // bottom edge walks the same rows and drops the records
                    // of rows off the detector: a row's share depends only
                    // on its own two boundaries, so this is exactly the
                    // reference's clamped range (cvp.cpp:197-201)
                    if (mode && !rows_inside) {
                        // preferably with virtual rows: the tile spans the
                        // unclamped row range, records of rows off the
                        // detector land in tile rows the forward's flush
                        // drops and the backward stages as zeros, and the
                        // brick walks the plain fast path (c3 P +1%, BP +2%;
                        // c2 P +3%, BP +2-5%); otherwise (tile too small) the
                        // clipping variant of the walk
                        const int tcu = max(n1 - n0 + 1, 0);
                        if (m1 >= m0 && tcu > 0 && ((r1u - r0u + 1) | 1) * tcu <= p.tile_cap) {
                            m0 = r0u;
                            m1 = r1u;
                        } else {
                            mode += 4;
                        }
                    }
                }
                // relaxed CutCentroid: one radius per voxel-cut where that
                // changes no record's 1/r^2 by more than 5e-6 relative: the
                // row-segment midpoints lie within h of the voxel centre, so
                // |d ln(1/r^2)| <= 2 (|dz|max + h) h / dmin^2
                if (CCR == 2 && mode != 0) {
                    const float hh = 0.5f * float(sc.a3);
                    const float zm = fmaxf(fabsf(zlo), fabsf(zhi)) + hh;
                    if (2.f * zm * hh <= 5e-6f * dmin * dmin) mode |= 8;
                }
                s.walk_mode = mode;
            }
            if (FWD) {
                // Forward accumulation is int32 fixed point (native ATOMS.ADD;
                // float shared atomics are CAS loops on sm_100). Bound on any
                // pixel's partial sum from this brick:
                //   |mu| <= mu_max;  inv_r2 <= 1/dmin^2 (r >= depth >= dmin);
                //   sum of cut areas in one detector column <= area of that
                //     column's wedge between depths dmin..dmax <= b1 dmax/f (dmax-dmin);
                //   sum over a column stack of one row's shares <= the row's
                //     z-window at the widest elevation depth <= b2 (dmax + diag/2)/f.
                // Scale 2^30 / bound keeps every partial inside int32 (float32
                // evaluation with 5% slack).
                const float bf = float(vc.b2_over_f);
                const float b1f = float(vc.b2_over_f) * b1_over_b2;  // b1 / f
                const float area = b1f * dmax * fmaxf(dmax - dmin, 1e-30f * dmax);
                const float zwin = bf * (dmax + 0.5f * diag);
                const float bound = s.mu_abs_max * fdiv_fp(area * zwin, dmin * dmin) * 1.05f;
                // (approximate reciprocal: q bound <= 2^30 (1 + 2^-22), far
                // inside int32 with the bound's 5% slack)
                const float q = (bound > 0.f && dmin > 0.f) ? 1073741824.f * fast_rcp(bound) : 0.f;
                // the fixed-point tile needs a finite brick and a normal
                // float32 scale; otherwise (NaN / Inf voxels, |mu| so small
                // that 2^30 / bound overflows) every record of this (brick,
                // view) takes the float-atomic path below, which propagates
                // NaN / Inf like the reference's double accumulation
                fixed_ok = !s.nonfinite && q > 0.f && q < 3.0e38f && q >= 1.17549435e-38f;
                s.qscale = fixed_ok ? q : 0.f;
            }
            const int tr = max(m1 - m0 + 1, 0), tc = max(n1 - n0 + 1, 0);
            const int stride = tr | 1;
            if (FWD && !fixed_ok && s.mu_abs_max == 0.f && !s.nonfinite) fixed_ok = true;  // all-zero brick
            s.tile_m0 = m0;
            s.tile_n0 = n0;
            s.tile_rows = tr;
            s.tile_cols = tc;
            s.tile_stride = stride;
            s.tile_ok = (tr > 0 && tc > 0 && stride * tc <= p.tile_cap && (!FWD || fixed_ok)) ? 1 : 0;
            const size_t vl = size_t(v - p.view_begin);
            s.img = FWD ? p.proj_out + vl * npx : const_cast<float*>(p.proj_in) + vl * npx;
            s.dimg = (FWD && s.det_g > 0.0) ? p.det_acc + vl * npx : nullptr;
            s.scale = p.scales + size_t(vc.scale_slot) * npx;
        };
        if (tid >= NT - BK) {
            // per-layer dz of this view (threads outside the G-phase; no
            // float64 per voxel-column in the V-phase)
            const int kk = tid - (NT - BK);
            const double zc64 = sc.minz + (k0 + kk + 0.5) * sc.a3;
            s.dz[kk] = EXACT ? float(zc64 - vc.s3) : float(zc64) - float(vc.s3);
        }
        // forward (no tile staging): the column loads are split over two
        // threads per column (slots 0-1 and 2-3), halving the dependent
        // L2-latency chain of the G-phase
        constexpr bool SPLIT_LOAD = FWD && 2 * NCOL <= NT;
        // (thread NCOL computes the footprint instead: column 0 keeps all slots)
        if (SPLIT_LOAD && tid > NCOL && tid < 2 * NCOL) {
            const int c = tid - NCOL;
            const int i = i0 + (c % BI), j = j0 + (c / BI);
            if (i < i1 && j < j1 && s.nonzero[c]) {
                // slots 2-3 unconditionally (no wait for the count: one L2
                // round trip; unused slots are never read)
                const size_t col = size_t(j) * sc.n1 + i;
                const size_t vl = size_t(v - p.t.v0);
                float4 ra[MAXC - 2], rb[MAXC - 2];
#pragma unroll
                for (int q = 2; q < MAXC; ++q) {
                    const size_t slot = (vl * MAXC + q) * p.t.ncols + col;
                    ra[q - 2] = __ldg(p.t.cutA + slot);
                    rb[q - 2] = __ldg(p.t.cutB + slot);
                }
#pragma unroll
                for (int q = 2; q < MAXC; ++q) {
                    s.cutA[q * NCOL + c] = ra[q - 2];
                    s.cutB[q * NCOL + c] = rb[q - 2];
                }
            }
        }
        if (tid < NCOL) {
            const int c = tid;
            const int i = i0 + (c % BI), j = j0 + (c / BI);
            int cnt = 0;
            // (a separate flag: the per-view cut count may be 0 for a column
            // whose cuts all fall off the detector in one view only)
            if (i < i1 && j < j1 && (!FWD || s.nonzero[c])) {
                // the column's cuts from the table (cut_table_kernel)
                const size_t col = size_t(j) * sc.n1 + i;
                const size_t vl = size_t(v - p.t.v0);
                const size_t base = vl * p.t.ncols + col;
                cnt = __ldg(p.t.count + base);
                if (SPLIT_LOAD) {
                    // slots 0-1 issued with the count (one L2 round trip)
                    float4 ra[2], rb[2];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const size_t slot = (vl * MAXC + q) * p.t.ncols + col;
                        ra[q] = __ldg(p.t.cutA + slot);
                        rb[q] = __ldg(p.t.cutB + slot);
                    }
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        s.cutA[q * NCOL + c] = ra[q];
                        s.cutB[q * NCOL + c] = rb[q];
                    }
                    if (c == 0)  // (thread NCOL computes the footprint)
                        for (int q = 2; q < min(cnt, MAXC); ++q) {
                            const size_t slot = (vl * MAXC + q) * p.t.ncols + col;
                            s.cutA[q * NCOL + c] = __ldg(p.t.cutA + slot);
                            s.cutB[q * NCOL + c] = __ldg(p.t.cutB + slot);
                        }
                } else {
                    const int nc = min(cnt, MAXC);
                    for (int q = 0; q < nc; ++q) {
                        const size_t slot = (vl * MAXC + q) * p.t.ncols + col;
                        s.cutA[q * NCOL + c] = __ldg(p.t.cutA + slot);
                        s.cutB[q * NCOL + c] = __ldg(p.t.cutB + slot);
                    }
                }
                const ColumnAnchor an = column_anchor<EXACT>(
                    vc.pp2, sc.minz + (k0 + 0.5) * sc.a3 - vc.s3, __ldg(p.t.Q0 + base), sc.a3);
                s.anchor[c] = make_int4(an.M0, __float_as_int(an.f0), __float_as_int(an.dh),
                                        __float_as_int(an.dl));
                s.rho2c[c] = __ldg(p.t.rho2c + base);
            }
            s.count[c] = cnt;
        } else if (SPLIT) {
            if (tid == NCOL) footprint();
            asm volatile("bar.sync 1, %0;" ::"r"(NT - NCOL) : "memory");
            tile_prologue(tid - NCOL, NT - NCOL);
        }
        if (!SPLIT && tid == (NCOL < NT ? NCOL : 0)) footprint();
        __syncthreads();
        const int tm0 = s.tile_m0, tn0 = s.tile_n0, trows = s.tile_rows, tcols = s.tile_cols;
        const int tstride = s.tile_stride;
        const uint32_t trm1 = uint32_t(trows - 1);
        const bool tile_ok = s.tile_ok != 0;
        // the brick's footprint misses the detector in this view: every
        // record would be clamped away (cvp.cpp:183-201), nothing to do
        if (trows == 0 || tcols == 0) continue;
        if (!SPLIT && !FWD && tile_ok) {
            tile_prologue(tid, NT);
            __syncthreads();
        }
        // ---- V-phase -----------------------------------------------------
        const float pp2f = float(vc.pp2);
        const float pp2h = pp2f + 0.5f;
        const float qs = FWD ? s.qscale : 0.f;
        // Forward, off-tile cuts: the view's image pointer is re-read from
        // shared memory inside that rare branch so no 64-bit address stays
        // live in the cut loop.
        const uint32_t img_slot = sbase + uint32_t(offsetof(Smem, img));
        const uint32_t dimg_slot = sbase + uint32_t(offsetof(Smem, dimg));
        const uint32_t detg_slot = sbase + uint32_t(offsetof(Smem, det_g));
        const uint32_t scale_slot = sbase + uint32_t(offsetof(Smem, scale));
        // Each lane carries NV voxels of one column through every cut (NV = NH
        // = 2: the cut record, tile test and loop control are shared
        // by the lane's voxels kk = lane and lane + 32).
        auto vphase = [&](auto mode_tag) {
        constexpr int MODE = decltype(mode_tag)::value;
        for (int ch = warp; ch < NCOL * NH / NV; ch += NWARP) {
            constexpr int NG = NH / NV;  // voxel groups per column
            const int c = ch / NG;
            const int hf0 = (ch % NG) * NV;
            const int cnt = lds_s32(sbase + uint32_t(offsetof(Smem, count)) + 4u * c);
            if (cnt == 0) continue;
            int4 a4;
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(a4.x), "=r"(a4.y), "=r"(a4.z), "=r"(a4.w)
                         : "r"(sbase + uint32_t(offsetof(Smem, anchor)) + 16u * c));
            // (+1/2 row shift of the walk folded into the anchor remainder and
            // pp2 once per column instead of per voxel)
            const ColumnAnchor an{a4.x, __int_as_float(a4.y) + 0.5f, __int_as_float(a4.z),
                                  __int_as_float(a4.w)};
            VoxState vs[NV];
            bool any_active = false;
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                VoxState& v = vs[t];
                const int kk = lane + 32 * (hf0 + t);
                const int k = k0 + kk;
                v.kvalid = k < k1;
                v.dz = lds_f32(sbase + uint32_t(offsetof(Smem, dz)) + 4u * kk);
                v.dz2e28 = v.dz * v.dz * 1e28f;  // rho2 < dz2e28  <=>  dz^2 > 1e-28 rho2
                v.vaddr = sbase + uint32_t(offsetof(Smem, vox)) + 4u * (c * MUS + kk);
                v.mu = FWD ? lds_f32(v.vaddr) : 0.f;
                v.active = v.kvalid && (!FWD || v.mu != 0.f);
                any_active |= v.active;
                float Mf;  // == float(v.Mi) exactly: not kept (one register per voxel)
                anchor_at(an, pp2h, float(kk), v.Mi, Mf, v.u0h, v.pmh);
                // forward: fixed-point scale folded into mu (the rare
                // off-tile walk re-reads mu itself, so only muq stays live)
                v.muq = v.mu * qs;
                v.inv_r2_fixed = per_row_r ? -1.f
                                           : fast_rcp(lds_f32(sbase + uint32_t(offsetof(Smem, rho2c)) + 4u * c) +
                                                      v.dz * v.dz);
                v.acc = 0.f;
            }
            // (one voxel group per column: the column's nonzero flag, which
            // zeroed its cut count in the G-phase, already guarantees an
            // active voxel)
            if (FWD && NG > 1 && !__any_sync(0xffffffffu, any_active)) continue;
            // One voxel-cut. TILE: the cut's column lies in the detector tile.
            // Every row with a nonzero share then lies inside the tile (the
            // footprint is conservative by >= 1 row, brick_footprint); rows
            // the walk visits beyond it carry share 0 exactly (both boundary
            // clamp-means saturate at +-h) and are clamped into the tile,
            // so the emits need no bounds branch. Otherwise (tile overflow,
            // column off the tile: warp-uniform, rare) emit to global memory.
            auto do_cut = [&](const CutRec& r, VoxState& v, auto tile_tag) {
                constexpr bool TILE = decltype(tile_tag)::value;
                // elevation correction unless the voxel sits in the source
                // plane (shw >= 0 always; shw = 0 makes it a no-op)
                const float sh = (corr && r.rho2 < v.dz2e28) ? r.shw : 0.f;
                const float uh = fmaf(v.dz, r.kc, v.u0h);
                const uint32_t cbase = tbase + 4u * uint32_t((r.n - tn0) * tstride);
                const float wA = FWD ? v.muq * r.A : r.A;
                float cut_acc = 0.f;
                if constexpr (!TILE) {
                    // off the tile (overflow, column outside it): rare, out of line
                    const float ca = offtile_walk<FWD, NR>(
                        r, v.Mi, float(v.Mi), uh, v.pmh, v.dz, h, sh, per_row_r ? 1 : 0, v.inv_r2_fixed,
                        rows, cols, FWD ? lds_f32(v.vaddr) : 0.f, reinterpret_cast<float*>(lds_u64(img_slot)),
                        reinterpret_cast<const float*>(lds_u64(scale_slot)),
                        reinterpret_cast<unsigned long long*>(lds_u64(dimg_slot)), lds_f64(detg_slot));
                    if (!FWD) v.acc = fmaf(wA, ca, v.acc);
                    return;
                }
                auto emit = [&](int m, float wr) {
                    // rows off the tile (either side) carry share 0: any
                    // in-tile slot will do, so one unsigned min clamps both
                    const uint32_t a = cbase + 4u * min(uint32_t(m - tm0), trm1);
                    if (FWD)
                        red_s32(a, __float2int_rn(wr * wA));
                    else
                        cut_acc = fmaf(lds_f32(a), wr, cut_acc);
                };
                walk_rows<true, decltype(emit)&, true, NR>(r, v.Mi, float(v.Mi), uh, v.pmh, v.dz, h, sh,
                                                           per_row_r, v.inv_r2_fixed, rows, emit);
                if (!FWD) v.acc = fmaf(wA, cut_acc, v.acc);
            };
            // fast walk (MODE 1 / 2): rows need no clamping and stay inside
            // the tile (2-row margin), so the addresses need no bound
            auto fast_cut = [&](const CutRec& r, VoxState& v) {
                // (fast mode: the elevation gate holds for every voxel-cut of
                // the brick, footprint())
                constexpr int NB = (MODE & 3) ? (MODE & 3) : 1;  // (MODE 0: unused)
                constexpr bool CLIP = (MODE & 4) != 0;  // rows off the detector: weight 0
                constexpr bool CUTR = (MODE & 8) != 0;  // relaxed: one radius per voxel-cut
                const float sh = corr ? r.shw : 0.f;
                const float uh = fmaf(v.dz, r.kc, v.u0h);
                // (unclipped: rows arrive biased by kRowBias, folded in here)
                constexpr bool RAW = !CLIP;
                const uint32_t cbase =
                    tbase + 4u * (uint32_t((r.n - tn0) * tstride - tm0) - (RAW ? uint32_t(kRowBias) : 0u));
                int nrow = 0;
                auto emit = [&](int m_in, float w) {
                    uint32_t a = cbase + 4u * uint32_t(m_in);
                    const int m = RAW ? m_in - kRowBias : m_in;
                    if (CLIP) {
                        // every on-detector row lies in the tile (2-row
                        // margin); the dropped ones write 0 to any tile slot
                        a = tbase + 4u * (uint32_t((r.n - tn0) * tstride) + min(uint32_t(m - tm0), trm1));
                        w = unsigned(m) < unsigned(rows) ? w : 0.f;
                    } else if (NB >= 2 && nrow == NB) {
                        a = tbase + 4u * min(uint32_t((r.n - tn0) * tstride + m - tm0),
                                             uint32_t((r.n - tn0) * tstride) + trm1);
                    }
                    ++nrow;
                    if (FWD)
                        red_s32(a, __float2int_rn(w));
                    else
                        v.acc = fmaf(lds_f32(a), w, v.acc);
                };
                const float ws = FWD ? v.muq * r.A : r.A;
                walk_rows_fast<NB, decltype(emit)&, CUTR, RAW>(r, v.Mi, uh, v.pmh, v.dz, h, sh, per_row_r,
                                                               v.inv_r2_fixed, ws, emit);
            };
            auto cut = [&](const CutRec& r) {
                if (tile_ok && unsigned(r.n - tn0) < unsigned(tcols)) {
                    // tile path: inactive voxels run too, with zero weight
                    // (forward: mu = 0) or a discarded accumulator (backward:
                    // k past the volume), so there is no per-voxel branch
                    if constexpr (MODE == 0) {
#pragma unroll
                        for (int t = 0; t < NV; ++t) do_cut(r, vs[t], std::true_type{});
                    } else {
#pragma unroll
                        for (int t = 0; t < NV; ++t) fast_cut(r, vs[t]);
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < NV; ++t)
                        if (vs[t].active) do_cut(r, vs[t], std::false_type{});
                }
            };
            if (any_active) {
                const int ncached = min(cnt, MAXC);
                // unrolled over the cut slots (constant record offsets, no
                // loop counter: c3 P +1-3%, BP +1%)
#pragma unroll
                for (int q = 0; q < MAXC; ++q) {
                    if (q >= ncached) break;
                    cut(load_cut(sbase, q * NCOL + c));
                }
                if (cnt > MAXC) {
                    // overflow (pixels much smaller than voxels): cuts >= MAXC
                    // recomputed out of line, kOverflowCap at a time
                    const int i = i0 + (c % BI), j = j0 + (c / BI);
                    CutRec extra[kOverflowCap];
                    for (int q0 = MAXC; q0 < cnt; q0 += kOverflowCap) {
                        overflow_cuts<EXACT>(&vc, sc, i, j, corr ? 1 : 0, q0, extra);
                        const int nx = min(cnt - q0, kOverflowCap);
                        for (int q = 0; q < nx; ++q) cut(extra[q]);
                    }
                }
            }
            if (!FWD) {
#pragma unroll
                for (int t = 0; t < NV; ++t)
                    if (vs[t].kvalid) sts_f32(vs[t].vaddr, lds_f32(vs[t].vaddr) + vs[t].acc);
            }
        }
        };
        {
            const int mode = s.walk_mode;
            auto dispatch = [&](auto cutr_tag) {
                constexpr int C = decltype(cutr_tag)::value;  // 0, or 8 (per-cut radius)
                const int m = mode & 7;
                if (m == 1)
                    vphase(std::integral_constant<int, 1 | C>{});
                else if (m == 5)
                    vphase(std::integral_constant<int, 5 | C>{});
                else if (m == 2)
                    vphase(std::integral_constant<int, 2 | C>{});
                else if (m == 6)
                    vphase(std::integral_constant<int, 6 | C>{});
                else if (m == 3)
                    vphase(std::integral_constant<int, 3 | C>{});
                else if (m == 7)
                    vphase(std::integral_constant<int, 7 | C>{});
                else
                    vphase(std::integral_constant<int, 0>{});
            };
            if (CCR == 2 && (mode & 8))
                dispatch(std::integral_constant<int, CCR == 2 ? 8 : 0>{});
            else
                dispatch(std::integral_constant<int, 0>{});
        }
        // ---- flush (forward) ----------------------------------------------
        // Lanes cover a power-of-two span of tile columns (coalesced float
        // atomics along an image row), warps and lane groups stride the rows:
        // no integer division in the loop.
        if (FWD && tile_ok) {
            __syncthreads();
            float* const view_img = s.img;
            unsigned long long* const view_dimg = s.dimg;
            const float inv_qs = qs > 0.f ? 1.f / qs : 0.f;
            const int span = tcols >= 32 ? 32 : tcols > 16 ? 32 : tcols > 8 ? 16 : tcols > 4 ? 8 : 4;
            const int lsh = 31 - __clz(span);             // log2(span)
            const int sub = lane >> lsh, rstep = NWARP << (5 - lsh);
            float* img = view_img + ptrdiff_t(tm0) * cols + tn0;  // (tm0 < 0: virtual rows)
            if (view_dimg) {
                // deterministic: the brick's (already order-independent)
                // int32 tile, rescaled to the launch-wide int64 quantum
                unsigned long long* dimg = view_dimg + ptrdiff_t(tm0) * cols + tn0;
                const double g = s.det_g;
                for (int c0 = 0; c0 < tcols; c0 += span) {
                    const int cc = c0 + (lane & (span - 1));
                    if (cc >= tcols) continue;
                    int* col = itile + cc * tstride;
                    for (int r = (warp << (5 - lsh)) + sub; r < trows; r += rstep) {
                        const int q = col[r];
                        if (q != 0) {
                            col[r] = 0;
                            if (unsigned(tm0 + r) < unsigned(rows))  // (virtual rows: dropped)
                                atomicAdd(dimg + size_t(r) * cols + cc,
                                          static_cast<unsigned long long>(
                                              __double2ll_rn(double(float(q) * inv_qs) * g)));
                        }
                    }
                }
            } else {
                for (int c0 = 0; c0 < tcols; c0 += span) {
                    const int cc = c0 + (lane & (span - 1));
                    if (cc >= tcols) continue;
                    int* col = itile + cc * tstride;
                    for (int r = (warp << (5 - lsh)) + sub; r < trows; r += rstep) {
                        const int q = col[r];
                        if (q != 0) {
                            col[r] = 0;
                            if (unsigned(tm0 + r) < unsigned(rows))  // (virtual rows: dropped)
                                atomicAdd(img + size_t(r) * cols + cc, float(q) * inv_qs);
                        }
                    }
                }
            }
        }
    }
    if (!FWD) {
        __syncthreads();
        for (int idx = tid; idx < NCOL * BK; idx += NT) {
            const int kk = idx / NCOL, c = idx % NCOL;
            const int i = i0 + (c % BI), j = j0 + (c / BI), kq = k0 + kk;
            if (i < i1 && j < j1 && kq < k1) {
                const size_t off = size_t(kq) * plane + size_t(j) * sc.n1 + i;
                const float val = s.vox[c * MUS + kk];
                if (p.tg.n > 0) {
                    // fused reduce-scatter: straight into the slab that owns
                    // plane kq (another GPU's memory over NVLink), while the
                    // other bricks are still computing; plain stores when this
                    // launch owns the region alone (one view group: each voxel
                    // is written by exactly one brick)
                    int t = 0;
                    while (t + 1 < p.tg.n && kq >= p.tg.plane_begin[t + 1]) ++t;
                    float* dst = p.tg.slab[t] + (off - size_t(p.tg.plane_begin[t]) * plane);
                    if (p.tg.store && !p.atomic_out)
                        *dst = p.accumulate ? *dst + val : val;
                    else
                        atomicAdd(dst, val);
                    continue;
                }
                float* dst = p.vol_out + off;
                if (p.atomic_out) {
                    atomicAdd(dst, val);
                } else {
                    const float out = p.accumulate ? *dst + val : val;
                    if (p.vol_out64)
                        p.vol_out64[off] = double(out);
                    else
                        *dst = out;
                }
            }
        }
    }
}

// Phase-2 scaling of the forward output (cvp.cpp:473-474), one streaming pass
// after all bricks have merged: out[v][px] *= scale[slot(v)][px].
__global__ void apply_scale_kernel(float* __restrict__ out, const float* __restrict__ scales,
                                   const ViewConst* __restrict__ views, int view_begin,
                                   size_t npx) {
    const int v = blockIdx.y;
    const float* sc = scales + size_t(views[view_begin + v].scale_slot) * npx;
    float* o = out + size_t(v) * npx;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < npx;
         i += size_t(gridDim.x) * blockDim.x)
        o[i] *= __ldg(sc + i);
}

// Deterministic forward: int64 fixed-point stack -> float32 output with the
// phase-2 scale (replaces apply_scale_kernel; *g == 0: the float atomics ran).
__global__ void det_finalize_kernel(float* __restrict__ out, const unsigned long long* __restrict__ acc,
                                    const double* __restrict__ g, const float* __restrict__ scales,
                                    const ViewConst* __restrict__ views, int view_begin, size_t npx) {
    const int v = blockIdx.y;
    const double gv = *g;
    const double inv = gv > 0.0 ? 1.0 / gv : 0.0;
    const float* sc = scales + size_t(views[view_begin + v].scale_slot) * npx;
    float* o = out + size_t(v) * npx;
    const unsigned long long* a = acc + size_t(v) * npx;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < npx;
         i += size_t(gridDim.x) * blockDim.x) {
        const float val = gv > 0.0 ? float(double(static_cast<long long>(a[i])) * inv) : o[i];
        o[i] = val * __ldg(sc + i);
    }
}

// Launch-wide int64 quantum of the deterministic forward: *g = 2^k with
// 2^k * bound <= 2^61, bound = max|mu| * factor >= any pixel's pre-scale sum
// (factor = voxel count * voxel volume / r_min^2: every voxel contributes at
// most its volume / r_min^2 to one pixel). Non-finite volume: *g = 0.
template <class T>
__global__ void det_absmax_kernel(const T* __restrict__ vol, size_t n, unsigned int* maxbits) {
    float m = 0.f;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const float v = fabsf(float(vol[i]));
        m = (v != v || m != m) ? __int_as_float(0x7fffffff) : fmaxf(m, v);  // NaN sticks
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float w = __shfl_xor_sync(0xffffffffu, m, o);
        m = (w != w || m != m) ? __int_as_float(0x7fffffff) : fmaxf(m, w);
    }
    // non-negative floats (and the canonical NaN above) order like their bits
    if ((threadIdx.x & 31) == 0) atomicMax(maxbits, __float_as_uint(m));
}

__global__ void det_scale_kernel(const unsigned int* maxbits, double factor, double* g) {
    const float m = __uint_as_float(*maxbits);
    const double bound = double(m) * factor;
    if (!isfinite(m) || !isfinite(bound)) {
        *g = 0.0;
    } else if (bound == 0.0) {
        *g = 1.0;
    } else {
        int e;
        frexp(0x1p61 / bound, &e);
        *g = ldexp(1.0, e - 1);  // power of two <= 2^61 / bound: exact 1/g
    }
}

// Per-pixel phase-2 factors (ScaleCache, cvp.cpp:264-302) in float64, stored
// as float32. Exact mode: 1/solid angle of the pixel seen from the source,
// evaluated as two Van Oosterom–Strackee triangles (cancellation-free; the
// reference's 2*pi - sum(acos) form carries ~1e-8 relative noise at C-arm
// pixel sizes). Cos mode: f^2 / (b1 b2 cos^3 theta) (cvp.cpp:288-292).
__device__ double tri_solid_angle(const double* a, const double* b, const double* c) {
    const double cx = b[1] * c[2] - b[2] * c[1];
    const double cy = b[2] * c[0] - b[0] * c[2];
    const double cz = b[0] * c[1] - b[1] * c[0];
    const double num = fabs(a[0] * cx + a[1] * cy + a[2] * cz);
    const double den = 1.0 + (a[0] * b[0] + a[1] * b[1] + a[2] * b[2]) +
                       (b[0] * c[0] + b[1] * c[1] + b[2] * c[2]) +
                       (c[0] * a[0] + c[1] * a[1] + c[2] * a[2]);
    return 2.0 * atan2(num, den);
}

__global__ void scale_image_kernel(double f, double pp1, double pp2, double b1, double b2, int rows,
                                   int cols, int exact, float* out, double* out64) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * cols) return;
    const int m = idx / cols, n = idx % cols;
    double s;
    if (!exact) {
        const double u = (n - pp1) * b1, w = (m - pp2) * b2;
        const double c = f / sqrt(u * u + w * w + f * f);
        s = f * f / (b1 * b2 * c * c * c);
    } else {
        const double u0 = (n - 0.5 - pp1) * b1, u1 = (n + 0.5 - pp1) * b1;
        const double w0 = (m - 0.5 - pp2) * b2, w1 = (m + 0.5 - pp2) * b2;
        double t[4][3] = {{u0, w0, f}, {u1, w0, f}, {u1, w1, f}, {u0, w1, f}};
        for (int q = 0; q < 4; ++q) {
            const double l = 1.0 / sqrt(t[q][0] * t[q][0] + t[q][1] * t[q][1] + t[q][2] * t[q][2]);
            t[q][0] *= l;
            t[q][1] *= l;
            t[q][2] *= l;
        }
        const double omega = tri_solid_angle(t[0], t[1], t[2]) + tri_solid_angle(t[0], t[2], t[3]);
        s = 1.0 / omega;
    }
    if (out) out[idx] = float(s);
    if (out64) out64[idx] = s;
}

// Single-voxel record dump through the device kernel's own geometry code
// (the bookkeeping view of collect_cut_records, cvp.cpp:652-689).
template <bool EXACT>
__global__ void cut_records_kernel(Scene sc, const ViewConst* views, int view, int i, int j, int k,
                                   int corr_opt, int per_row_r, int clamp, int cap, int* rows_out,
                                   int* cols_out, double* vol_out, double* inv_out, int* n_out,
                                   int* err) {
    const ViewConst vc = views[view];
    const double zc64 = sc.minz + (k + 0.5) * sc.a3;
    const double dz64 = zc64 - vc.s3;
    const float dz = EXACT ? float(dz64) : float(zc64) - float(vc.s3);
    const float h = float(0.5 * sc.a3);
    const bool corr = corr_opt != 0;
    int count = 0;
    // records report (volume, inv_r2); the walk hands share * inv_r2, so the
    // debug path re-derives inv_r2 = 1 / (rho2 + zr^2) by walking twice:
    // once with a unit-area cut to collect share * inv_r2 and the volume.
    int cur_n = 0;
    float cur_A = 0.f;
    ColumnRec col;
    const int st = column_cuts<EXACT>(vc, sc, i, j, clamp != 0, corr, col, [&](const CutRec&) {});
    if (st < 0) {
        *err = kDevSourcePlane;
        *n_out = 0;
        return;
    }
    int Mi;
    float Mf, u0, pm;
    voxel_anchor<EXACT>(vc.pp2, dz64, dz, col.Q0, Mi, Mf, u0, pm);
    const float inv_r2_fixed = per_row_r ? -1.f : fast_rcp(col.rho2c + dz * dz);
    column_cuts<EXACT>(vc, sc, i, j, clamp != 0, corr, col, [&](const CutRec& r) {
        const float shc = (corr && dz * dz > r.rho2 * 1e-28f) ? r.shw : 0.f;
        const float uh = fmaf(dz, r.kc, u0 + 0.5f), pmh = pm + 0.5f;
        cur_n = r.n;
        cur_A = r.A;
        // pass 1: share * inv_r2; pass 2 (fixed inv_r2 = 1): share alone
        float wr[64], sh[64];
        int ms[64], nrec = 0;
        auto take = [&](int m, float v) {
            if (nrec < 64) {
                ms[nrec] = m;
                wr[nrec] = v;
            }
            ++nrec;
        };
        int nrec2 = 0;
        auto take2 = [&](int, float v) {
            if (nrec2 < 64) sh[nrec2] = v;
            ++nrec2;
        };
        if (clamp) {
            walk_rows<true>(r, Mi, Mf, uh, pmh, dz, h, shc, per_row_r != 0, inv_r2_fixed,
                            sc.rows, take);
            walk_rows<true>(r, Mi, Mf, uh, pmh, dz, h, shc, false, 1.f, sc.rows, take2);
        } else {
            walk_rows<false>(r, Mi, Mf, uh, pmh, dz, h, shc, per_row_r != 0, inv_r2_fixed,
                             sc.rows, take);
            walk_rows<false>(r, Mi, Mf, uh, pmh, dz, h, shc, false, 1.f, sc.rows, take2);
        }
        for (int t = 0; t < nrec && t < 64; ++t) {
            if (count < cap) {
                rows_out[count] = ms[t];
                cols_out[count] = cur_n;
                vol_out[count] = double(cur_A) * sh[t];
                inv_out[count] = sh[t] > 0.f ? double(wr[t]) / sh[t] : 0.0;
            }
            ++count;
        }
    });
    *n_out = count;
}

template <bool EXACT, bool FWD, bool CORR, int CCR, int NR>
cudaError_t launch_variant(const CvpParams& p, dim3 grid, int dyn, cudaStream_t stream) {
    cudaError_t e = cudaFuncSetAttribute(cvp_brick_kernel<EXACT, FWD, CORR, CCR, NR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    if (e != cudaSuccess) return e;
    cvp_brick_kernel<EXACT, FWD, CORR, CCR, NR><<<grid, NT, dyn, stream>>>(p);
    return cudaGetLastError();
}

// Three straight-line rows only for the reference-default options (elevation
// correction, CutCentroid radius); other option sets walk two.
template <bool EXACT, bool FWD>
cudaError_t launch_opts(const CvpParams& p, dim3 grid, int dyn, bool tall, cudaStream_t stream) {
    if (p.corr) {
        if (p.per_row_r == 2)
            return tall ? launch_variant<EXACT, FWD, true, 2, 3>(p, grid, dyn, stream)
                        : launch_variant<EXACT, FWD, true, 2, 2>(p, grid, dyn, stream);
        return p.per_row_r ? (tall ? launch_variant<EXACT, FWD, true, 1, 3>(p, grid, dyn, stream)
                                   : launch_variant<EXACT, FWD, true, 1, 2>(p, grid, dyn, stream))
                           : launch_variant<EXACT, FWD, true, 0, 2>(p, grid, dyn, stream);
    }
    if (p.per_row_r == 2) return launch_variant<EXACT, FWD, false, 2, 2>(p, grid, dyn, stream);
    return p.per_row_r ? launch_variant<EXACT, FWD, false, 1, 2>(p, grid, dyn, stream)
                       : launch_variant<EXACT, FWD, false, 0, 2>(p, grid, dyn, stream);
}

// The per-(view, column) cut table (BandCutter + compute_cuts + fill_cut_info,
// cvp.cpp:73-157, via column_cuts): one thread per (view, column), consecutive
// threads on consecutive columns so the SoA stores coalesce.
template <bool EXACT>
__global__ void cut_table_kernel(Scene sc, const ViewConst* views, CutTable t, int corr, int* err) {
    const size_t ncols = size_t(t.ncols);
    const size_t total = ncols * t.nv;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const size_t col = idx % ncols, vl = idx / ncols;
        const int i = int(col % sc.n1), j = int(col / sc.n1);
        ColumnRec rec;
        int cnt = 0;
        cnt = column_cuts<EXACT>(views[t.v0 + vl], sc, i, j, true, corr != 0, rec, [&](const CutRec& r) {
            if (cnt < MAXC) {
                const size_t slot = (vl * MAXC + cnt) * ncols + col;
                t.cutA[slot] = make_float4(r.A, r.g, r.rho2, r.shw);
                t.cutB[slot] = make_float4(r.kc, r.tr_a, r.tr_b, __int_as_float(r.n));
            }
            ++cnt;
        });
        if (cnt < 0) {
            atomicOr(err, kDevSourcePlane);
            cnt = 0;
        }
        t.count[idx] = cnt;
        t.Q0[idx] = rec.Q0;
        t.rho2c[idx] = rec.rho2c;
    }
}

cudaError_t run_cut_table(const Scene& sc, const ViewConst* views, const CutTable& t, int exact,
                          int corr, int* err, cudaStream_t stream) {
    const size_t total = size_t(t.ncols) * t.nv;
    const int blocks = int(std::min<size_t>((total + 255) / 256, 148 * 64));
    (void)exact;  // float64 world quantities in both precisions (api.cpp run_cvp)
    cut_table_kernel<true><<<blocks, 256, 0, stream>>>(sc, views, t, corr, err);
    return cudaGetLastError();
}

// Carve a cut table for nv views out of the scratch block.
CutTable cut_table_layout(void* mem, int ncols, int v0, int nv) {
    CutTable t;
    const size_t n = size_t(ncols) * nv;
    unsigned char* m = static_cast<unsigned char*>(mem);
    t.cutA = reinterpret_cast<float4*>(m);
    m += sizeof(float4) * n * MAXC;
    t.cutB = reinterpret_cast<float4*>(m);
    m += sizeof(float4) * n * MAXC;
    t.Q0 = reinterpret_cast<double*>(m);
    m += sizeof(double) * n;
    t.count = reinterpret_cast<int*>(m);
    m += sizeof(int) * n;
    t.rho2c = reinterpret_cast<float*>(m);
    t.v0 = v0;
    t.nv = nv;
    t.ncols = ncols;
    return t;
}

// Largest tile (odd row stride x columns) any brick needs under any view.
__global__ void tile_need_kernel(Scene sc, const ViewConst* views, int n_views, int* need) {
    const int nbi = (sc.n1 + BI - 1) / BI, nbj = (sc.n2 + BJ - 1) / BJ, nbk = (sc.n3 + BK - 1) / BK;
    const long long total = (long long)nbi * nbj * nbk * n_views;
    int best = 0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        long long b = t / n_views;
        const int v = int(t % n_views);
        const int bi = int(b % nbi);
        b /= nbi;
        const int bj = int(b % nbj), bk = int(b / nbj);
        const int i0 = bi * BI, j0 = bj * BJ, k0 = bk * BK;
        int m0, m1, n0, n1;
        brick_footprint(views[v], sc, i0, min(i0 + BI, sc.n1), j0, min(j0 + BJ, sc.n2), k0,
                        min(k0 + BK, sc.n3), m0, m1, n0, n1);
        const int tr = max(m1 - m0 + 1, 0), tc = max(n1 - n0 + 1, 0);
        best = max(best, (tr | 1) * tc);
    }
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMax(need, best);
}

}  // namespace

cudaError_t CVP_PUB(launch_cvp_tile_need)(const Scene& sc, const ViewConst* views, int n_views,
                                          int* d_need, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(d_need, 0, sizeof(int), stream);
    if (e != cudaSuccess || n_views <= 0) return e;
    tile_need_kernel<<<148 * 4, 256, 0, stream>>>(sc, views, n_views, d_need);
    return cudaGetLastError();
}

namespace {
// Shared-memory budget per CTA for three resident CTAs per SM (228 KB SM
// carve-out, 1 KB reserved per CTA) and the hard cap for the detector tile.
constexpr int kSmemBudget3 = (228 * 1024) / CVP_MINB - 1024;
constexpr int kTileCapMax = 16384;
}  // namespace

cudaError_t CVP_PUB(launch_cvp)(const CvpLaunch& L, cudaStream_t stream) {
    const Scene& sc = L.sc;
    if (L.view_count <= 0) return cudaSuccess;
    // size the detector tile to the scene's largest brick footprint; three
    // CTAs per SM when it fits the budget, otherwise two with a larger tile
    int tile_cap = std::min(std::max(L.tile_need, 1), kTileCapMax);
    const int fit3 = (kSmemBudget3 - int(sizeof(Smem))) / int(sizeof(float));
    if (tile_cap <= fit3) tile_cap = fit3;
    const int dyn = int(sizeof(Smem)) + tile_cap * int(sizeof(float));
    const int nbricks = ((sc.n1 + BI - 1) / BI) * ((sc.n2 + BJ - 1) / BJ) * ((sc.n3 + BK - 1) / BK);

    CvpParams p;
    p.sc = sc;
    p.views = L.views;
    p.scales = L.scales;
    p.corr = L.elevation_correction;
    // relaxed precision + CutCentroid: the per-voxel-cut radius where allowed
    p.per_row_r = L.cut_centroid ? (L.relaxed && L.cut_radius_ok ? 2 : 1) : 0;
    p.h = float(0.5 * sc.a3);
    p.tile_cap = tile_cap;
    // CVPB_NO_TILE=1: every record takes the global (float-atomic / direct
    // gather) path, which otherwise only tile-overflow bricks use (tests)
    if (const char* e = std::getenv("CVPB_NO_TILE"))
        if (e[0] == '1') p.tile_cap = 0;
    p.err = L.err;
    p.tg = L.targets;

    // view chunks whose cut table fits the scratch block
    const int ncols = sc.n1 * sc.n2;
    const size_t per_view = size_t(ncols) * kCutTableBytes;
    const bool resident = L.cut_table_valid && L.view_begin >= L.table_v0 &&
                          L.view_begin + L.view_count <= L.table_v0 + L.table_nv;
    const int chunk = resident ? L.view_count
                               : int(std::min<size_t>(size_t(L.view_count),
                                                      L.cut_table ? L.cut_table_bytes / per_view : 0));
    if (chunk < 1) return cudaErrorMemoryAllocation;
    static_assert(kCutTableBytes == 2 * MAXC * sizeof(float4) + sizeof(double) + sizeof(int) + sizeof(float),
                  "cut table layout");
    const size_t npx = size_t(sc.rows) * sc.cols;
    const size_t nvox = size_t(sc.n1) * sc.n2 * sc.n3;

    cudaError_t e;
    const bool det = L.forward && L.det_acc && L.det_g && L.det_maxbits;
    if (L.forward) {
        e = cudaMemsetAsync(L.proj_out, 0, sizeof(float) * npx * L.view_count, stream);
        if (e != cudaSuccess) return e;
    }
    if (det) {
        // the quantum from max |mu| over the input (the float64 host volume
        // when the first chunk reads it in place)
        e = cudaMemsetAsync(L.det_acc, 0, sizeof(unsigned long long) * npx * L.view_count, stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(L.det_maxbits, 0, sizeof(unsigned int), stream);
        if (e != cudaSuccess) return e;
        if (L.vol_in64)
            det_absmax_kernel<double><<<148 * 8, 256, 0, stream>>>(L.vol_in64, nvox, L.det_maxbits);
        else
            det_absmax_kernel<float><<<148 * 8, 256, 0, stream>>>(L.vol_in, nvox, L.det_maxbits);
        det_scale_kernel<<<1, 1, 0, stream>>>(L.det_maxbits, 2.0 * L.det_factor, L.det_g);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    p.det_acc = nullptr;
    p.det_g = det ? L.det_g : nullptr;
    for (int c0 = 0; c0 < L.view_count; c0 += chunk) {
        const int cn = std::min(chunk, L.view_count - c0);
        const int cv0 = L.view_begin + c0;
        const bool first = c0 == 0, last = c0 + cn == L.view_count;
        if (resident) {
            p.t = cut_table_layout(L.cut_table, ncols, L.table_v0, L.table_nv);
        } else {
            p.t = cut_table_layout(L.cut_table, ncols, cv0, cn);
            e = run_cut_table(sc, L.views, p.t, L.exact, L.elevation_correction, L.err, stream);
            if (e != cudaSuccess) return e;
        }
        // Enough CTAs to fill 148 SMs x 2 resident: split views into groups
        // when the volume has few bricks (c1: 32 bricks). Deterministic mode
        // keeps one group so the backward accumulation order is fixed.
        int groups = 1;
        const int target = 148 * 2 * 2;
        if (!L.deterministic && nbricks < target) groups = std::min(cn, (target + nbricks - 1) / nbricks);
        const int per = (cn + groups - 1) / groups;
        groups = (cn + per - 1) / per;
        p.view_begin = cv0;
        p.view_count = cn;
        p.views_per_group = per;
        p.vol_in = L.vol_in;
        p.vol_out = L.vol_out;
        p.vol_in64 = first ? L.vol_in64 : nullptr;   // later chunks read the float32 copy
        p.vol_copy = first ? L.vol_copy : nullptr;
        p.proj_in = L.proj_in ? L.proj_in + size_t(c0) * npx : nullptr;
        p.proj_out = L.proj_out ? L.proj_out + size_t(c0) * npx : nullptr;
        p.det_acc = det ? L.det_acc + size_t(c0) * npx : nullptr;
        p.accumulate = first ? L.accumulate : 1;
        p.atomic_out = groups > 1 ? 1 : 0;
        // zero-copy float64 output on the last chunk (atomic view groups: convert after)
        p.vol_out64 = (last && groups == 1) ? L.vol_out64 : nullptr;
        if (!L.forward && groups > 1 && !p.accumulate && L.targets.n == 0) {
            e = cudaMemsetAsync(L.vol_out, 0, sizeof(float) * nvox, stream);
            if (e != cudaSuccess) return e;
        }
        if (!L.forward && groups > 1 && !p.accumulate && L.targets.n > 0 && L.targets.store) {
            // several view groups add with atomics: the overwrite semantics
            // of store mode start from zeroed regions (peer memory included)
            for (int t = 0; t < L.targets.n; ++t) {
                const size_t cnt = size_t(L.targets.plane_begin[t + 1] - L.targets.plane_begin[t]) *
                                   size_t(sc.n1) * sc.n2;
                if (cnt == 0) continue;
                e = cudaMemsetAsync(L.targets.slab[t], 0, sizeof(float) * cnt, stream);
                if (e != cudaSuccess) return e;
            }
        }
        dim3 grid(nbricks, groups);
        // (float64 world quantities in both precisions: EXACT geometry always)
        e = L.forward ? launch_opts<true, true>(p, grid, dyn, L.tall_voxels, stream)
                      : launch_opts<true, false>(p, grid, dyn, L.tall_voxels, stream);
        if (e != cudaSuccess) return e;
        if (!L.forward && last && L.vol_out64 && !p.vol_out64 && L.targets.n == 0) {
            e = launch_f32_to_f64(L.vol_out, L.vol_out64, nvox, stream);
            if (e != cudaSuccess) return e;
        }
    }
    if (L.forward) {
        const int bx = int(std::min<size_t>((npx + 255) / 256, 64));
        if (det)
            det_finalize_kernel<<<dim3(bx, L.view_count), 256, 0, stream>>>(
                L.proj_out, L.det_acc, L.det_g, L.scales, L.views, L.view_begin, npx);
        else
            apply_scale_kernel<<<dim3(bx, L.view_count), 256, 0, stream>>>(L.proj_out, L.scales, L.views,
                                                                           L.view_begin, npx);
        return cudaGetLastError();
    }
    return cudaSuccess;
}

#if !defined(CVP_CFG_B) && !defined(CVP_CFG_C)
cudaError_t launch_cut_table(const CvpLaunch& L, cudaStream_t stream) {
    const int ncols = L.sc.n1 * L.sc.n2;
    if (L.view_count <= 0) return cudaSuccess;
    if (!L.cut_table || size_t(ncols) * kCutTableBytes * L.view_count > L.cut_table_bytes)
        return cudaErrorMemoryAllocation;
    return run_cut_table(L.sc, L.views, cut_table_layout(L.cut_table, ncols, L.view_begin, L.view_count),
                         L.exact, L.elevation_correction, L.err, stream);
}

namespace {
// one CTA row per view: sum of the per-column cut counts (view_seconds weights)
__global__ void view_work_kernel(const int* __restrict__ count, int ncols, int vl0,
                                 unsigned long long* work) {
    const int v = blockIdx.y;
    const int* c = count + size_t(vl0 + v) * ncols;
    unsigned long long s = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncols; i += gridDim.x * blockDim.x)
        s += unsigned(max(c[i], 0));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(work + v, s);
}
}  // namespace

cudaError_t launch_view_work(void* cut_table, int ncols, int table_v0, int table_nv, int view_begin,
                             int view_count, unsigned long long* work, cudaStream_t stream) {
    if (view_count <= 0) return cudaSuccess;
    if (!cut_table || view_begin < table_v0 || view_begin + view_count > table_v0 + table_nv)
        return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(work, 0, sizeof(unsigned long long) * view_count, stream);
    if (e != cudaSuccess) return e;
    const CutTable t = cut_table_layout(cut_table, ncols, table_v0, table_nv);
    const int bx = std::min((ncols + 255) / 256, 16);
    view_work_kernel<<<dim3(bx, view_count), 256, 0, stream>>>(t.count, ncols, view_begin - table_v0, work);
    return cudaGetLastError();
}

cudaError_t launch_scale_image(double f, double pp1, double pp2, double b1, double b2, int rows,
                               int cols, int exact, float* out, double* out64, cudaStream_t stream) {
    const int n = rows * cols;
    scale_image_kernel<<<(n + 255) / 256, 256, 0, stream>>>(f, pp1, pp2, b1, b2, rows, cols, exact,
                                                           out, out64);
    return cudaGetLastError();
}

cudaError_t launch_cut_records(const Scene& sc, const ViewConst* views, int view, int i, int j,
                               int k, int exact, int corr, int per_row_r, int clamp, int cap,
                               int* rows, int* cols, double* vol, double* inv, int* n_out, int* err,
                               cudaStream_t stream) {
    (void)exact;
    cut_records_kernel<true><<<1, 1, 0, stream>>>(sc, views, view, i, j, k, corr, per_row_r, clamp,
                                                  cap, rows, cols, vol, inv, n_out, err);
    return cudaGetLastError();
}
#endif  // shape-independent entry points

}  // namespace cvpb
