// Device-resident vector operations for CGLS (solver.cpp:15-106): compensated
// float64 dot products of float32 vectors, axpy / xpby updates and the finite
// check. All are HBM-streaming kernels sized as a multiple of the 148 SMs.
#include <cmath>

#include "kernels.hpp"

namespace cvpb {

namespace {

constexpr int kDotBlocks = 148 * 4;
constexpr int kThreads = 256;

// Per-thread Kahan accumulation of exact float32 x float32 products in
// float64 (dot_kahan, solver.cpp:15-24), then a pairwise block reduction.
__global__ void dot_kernel(const float* __restrict__ a, const float* __restrict__ b, size_t n,
                           double* partials) {
    double sum = 0.0, c = 0.0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    // float4 main body when both pointers are 16-byte aligned
    const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
    if (vec) {
        const size_t n4 = n / 4;
        const float4* a4 = reinterpret_cast<const float4*>(a);
        const float4* b4 = reinterpret_cast<const float4*>(b);
        for (size_t q = i; q < n4; q += stride) {
            const float4 x = __ldg(a4 + q), y = __ldg(b4 + q);
            const double p = double(x.x) * y.x + double(x.y) * y.y + double(x.z) * y.z +
                             double(x.w) * y.w;
            const double yk = p - c;
            const double t = sum + yk;
            c = (t - sum) - yk;
            sum = t;
        }
        i = n4 * 4 + i;
    }
    for (; i < n; i += stride) {
        const double p = double(a[i]) * double(b[i]);
        const double yk = p - c;
        const double t = sum + yk;
        c = (t - sum) - yk;
        sum = t;
    }
    double v = sum - c;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __shared__ double ws[kThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) s += ws[w];
        partials[blockIdx.x] = s;
    }
}

__global__ void axpy_kernel(double alpha, const float* __restrict__ x, float* __restrict__ y,
                            size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride)
        y[i] = float(double(y[i]) + alpha * double(x[i]));
}

__global__ void xpby_kernel(const float* __restrict__ s, double beta, float* __restrict__ p,
                            size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride)
        p[i] = float(double(s[i]) + beta * double(p[i]));
}

__global__ void finite_kernel(const float* __restrict__ x, size_t n, int* flag) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    bool bad = false;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride)
        bad |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 0);
}

__global__ void f64_to_f32_kernel(const double* __restrict__ in, float* __restrict__ out, size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride)
        out[i] = float(in[i]);
}

__global__ void f32_to_f64_kernel(const float* __restrict__ in, double* __restrict__ out, size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride)
        out[i] = double(in[i]);
}

// SART (Andersen & Kak) pieces: r = (b - Ax) / (A 1) where A 1 > eps, else 0;
// x += lambda * (A^T r) / (A^T 1) where A^T 1 > eps, optionally clamped >= 0.
__global__ void sart_residual_kernel(const float* __restrict__ b, const float* __restrict__ ax,
                                     const float* __restrict__ rowsum, float* __restrict__ out,
                                     size_t n, float eps) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
        const float w = rowsum[i];
        out[i] = w > eps ? (b[i] - ax[i]) / w : 0.f;
    }
}

__global__ void sart_update_kernel(float* __restrict__ x, const float* __restrict__ corr,
                                   const float* __restrict__ colsum, float lambda, int nonneg,
                                   size_t n, float eps) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
        const float w = colsum[i];
        float v = x[i] + (w > eps ? lambda * corr[i] / w : 0.f);
        if (nonneg) v = fmaxf(v, 0.f);
        x[i] = v;
    }
}

// ---- fused, device-resident CGLS vector phase (solver.cpp:55-106) ---------
// The scalars (gamma, alpha, beta, the residual history) never leave the
// device inside an iteration: one single-warp kernel folds the dot partials in
// a fixed order (bit-reproducible) and updates CgState; the streaming kernels
// read alpha / beta from it and do nothing once the recurrence has stopped.

__device__ __forceinline__ double fold_partials(const double* __restrict__ p, int np) {
    // one warp, fixed lane order, Kahan per lane then a fixed butterfly
    double sum = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < np; i += 32) {
        const double y = p[i] - c;
        const double t = sum + y;
        c = (t - sum) - y;
        sum = t;
    }
    double v = sum - c;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void cg_scalar_kernel(int mode, const double* __restrict__ p1,
                                 const double* __restrict__ p2, int np, CgState* st, double* hist,
                                 int it) {
    const double a = fold_partials(p1, np);
    const double b = mode == 3 ? fold_partials(p2, np) : 0.0;
    if (threadIdx.x != 0) return;
    switch (mode) {
    case 0:  // ||b||: history entry 0
        st->status = 0;
        st->iteration = 0;
        hist[0] = sqrt(a);
        break;
    case 1:  // gamma = s.s after the first adjoint
        st->gamma = a;
        break;
    case 2:  // qq = q.q -> alpha (or the reference's two early exits)
        st->finite = 1;
        if (st->status != 0) break;
        if (st->gamma == 0.0) {
            st->status = kCgFlat;  // normal equations satisfied: history stays flat
            st->iteration = it;
        } else if (a == 0.0) {
            st->status = kCgBreakdown;
            st->iteration = it;
        } else {
            st->alpha = st->gamma / a;
        }
        break;
    case 3:  // gamma_new = s.s -> beta, rr = r.r -> history, finite check
        if (st->status == 0) {
            st->beta = a / st->gamma;
            st->gamma = a;
            if (!st->finite) {
                st->status = kCgDiverged;
                st->iteration = it;
            }
            hist[it] = sqrt(b);
        } else if (st->status == kCgFlat) {
            hist[it] = hist[it - 1];
        }
        break;
    }
}

// x += alpha p (n), r -= alpha q (m); partials of r.r (updated r) and the
// finite check of both iterates, in one pass.
__global__ void cg_update_kernel(const CgState* __restrict__ st, float* __restrict__ x,
                                 const float* __restrict__ p, size_t n, float* __restrict__ r,
                                 const float* __restrict__ q, size_t m, double* partials,
                                 int* finite) {
    if (st->status != 0) return;
    const double alpha = st->alpha;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    const size_t t0 = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    bool bad = false;
    for (size_t i = t0; i < n; i += stride) {
        const float v = float(double(x[i]) + alpha * double(__ldg(p + i)));
        x[i] = v;
        bad |= !isfinite(v);
    }
    double sum = 0.0, c = 0.0;
    for (size_t i = t0; i < m; i += stride) {
        const float v = float(double(r[i]) - alpha * double(__ldg(q + i)));
        r[i] = v;
        bad |= !isfinite(v);
        const double y = double(v) * double(v) - c;
        const double t = sum + y;
        c = (t - sum) - y;
        sum = t;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(finite, 0);
    double v = sum - c;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __shared__ double ws[kThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) s += ws[w];
        partials[blockIdx.x] = s;
    }
}

__global__ void cg_xpby_kernel(const CgState* __restrict__ st, const float* __restrict__ s,
                               float* __restrict__ p, size_t n) {
    if (st->status != 0) return;
    const double beta = st->beta;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride)
        p[i] = float(double(__ldg(s + i)) + beta * double(p[i]));
}

inline int grid_for(size_t n) {
    const size_t blocks = (n + kThreads - 1) / kThreads;
    return int(blocks < size_t(148 * 16) ? (blocks > 0 ? blocks : 1) : 148 * 16);
}

}  // namespace

int dot_partials_count() { return kDotBlocks; }

cudaError_t launch_dot(const float* a, const float* b, size_t n, double* d_partials,
                       int n_partials, cudaStream_t stream) {
    if (n_partials < kDotBlocks) return cudaErrorInvalidValue;
    dot_kernel<<<kDotBlocks, kThreads, 0, stream>>>(a, b, n, d_partials);
    return cudaGetLastError();
}

cudaError_t launch_cg_scalar(int mode, const double* p1, const double* p2, CgState* st,
                             double* hist, int it, cudaStream_t stream) {
    cg_scalar_kernel<<<1, 32, 0, stream>>>(mode, p1, p2, kDotBlocks, st, hist, it);
    return cudaGetLastError();
}

cudaError_t launch_cg_update(const CgState* st, float* x, const float* p, size_t n, float* r,
                             const float* q, size_t m, double* partials, int* finite,
                             cudaStream_t stream) {
    cg_update_kernel<<<kDotBlocks, kThreads, 0, stream>>>(st, x, p, n, r, q, m, partials, finite);
    return cudaGetLastError();
}

cudaError_t launch_cg_xpby(const CgState* st, const float* s, float* p, size_t n,
                           cudaStream_t stream) {
    cg_xpby_kernel<<<grid_for(n), kThreads, 0, stream>>>(st, s, p, n);
    return cudaGetLastError();
}

cudaError_t launch_axpy(double alpha, const float* x, float* y, size_t n, cudaStream_t stream) {
    axpy_kernel<<<grid_for(n), kThreads, 0, stream>>>(alpha, x, y, n);
    return cudaGetLastError();
}

cudaError_t launch_xpby(const float* s, double beta, float* p, size_t n, cudaStream_t stream) {
    xpby_kernel<<<grid_for(n), kThreads, 0, stream>>>(s, beta, p, n);
    return cudaGetLastError();
}

cudaError_t launch_all_finite(const float* x, size_t n, int* d_flag, cudaStream_t stream) {
    finite_kernel<<<grid_for(n), kThreads, 0, stream>>>(x, n, d_flag);
    return cudaGetLastError();
}

cudaError_t launch_sart_residual(const float* b, const float* ax, const float* rowsum, float* out,
                                 size_t n, float eps, cudaStream_t stream) {
    sart_residual_kernel<<<grid_for(n), kThreads, 0, stream>>>(b, ax, rowsum, out, n, eps);
    return cudaGetLastError();
}

cudaError_t launch_sart_update(float* x, const float* corr, const float* colsum, float lambda,
                               int nonneg, size_t n, float eps, cudaStream_t stream) {
    sart_update_kernel<<<grid_for(n), kThreads, 0, stream>>>(x, corr, colsum, lambda, nonneg, n, eps);
    return cudaGetLastError();
}

cudaError_t launch_f64_to_f32(const double* in, float* out, size_t n, cudaStream_t stream) {
    f64_to_f32_kernel<<<grid_for(n), kThreads, 0, stream>>>(in, out, n);
    return cudaGetLastError();
}

cudaError_t launch_f32_to_f64(const float* in, double* out, size_t n, cudaStream_t stream) {
    f32_to_f64_kernel<<<grid_for(n), kThreads, 0, stream>>>(in, out, n);
    return cudaGetLastError();
}

}  // namespace cvpb
