// Siddon-K ray-driven projector pair for sm_100a.
//
// Reference: /root/reference/proj/src/siddon.cpp — traverse (:37-98),
// DetectorPlane (:135-150), project_siddon_k_into (:166-249),
// backproject_siddon_k_into (:259-313).
//
// One thread per (pixel, view) walks its K x K sub-rays with the reference's
// incremental parametric traversal in float64 (ties advance every tying axis;
// half-open voxel intervals), reading attenuation through the read-only path.
// The forward restricts traversal to the tight box of nonzero voxels exactly
// like the reference (:182-211); the backward scatters w * chord with device
// atomics (the reference's `omp atomic`, :299-304). The value type T is float
// for the device API and double for the reference-facing host path, where
// Siddon is the float64 ground truth the reference makes it (its unit tests
// pin chords and linearity at 1e-9 / 1e-12).
#include <cfloat>

#include "kernels.hpp"

namespace cvpb {

namespace {

struct Box {
    double lo[3], a[3];
    int i0[3], n[3];
};

template <class Emit>
__device__ __forceinline__ void traverse(const Box& b, const double s[3], const double d[3],
                                         double dlen, Emit&& emit) {
    double t0 = 0.0, t1 = INFINITY;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const double hi = b.lo[ax] + b.a[ax] * b.n[ax];
        if (d[ax] == 0.0) {
            if (s[ax] < b.lo[ax] || s[ax] >= hi) return;
        } else {
            double ta = (b.lo[ax] - s[ax]) / d[ax];
            double tb = (hi - s[ax]) / d[ax];
            if (ta > tb) {
                const double x = ta;
                ta = tb;
                tb = x;
            }
            t0 = fmax(t0, ta);
            t1 = fmin(t1, tb);
        }
    }
    if (!(t0 < t1)) return;
    int idx[3], step[3];
    double tnext[3], tdelta[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const double pos = s[ax] + t0 * d[ax];
        idx[ax] = min(max(int(floor((pos - b.lo[ax]) / b.a[ax])), 0), b.n[ax] - 1);
        if (d[ax] > 0.0) {
            step[ax] = 1;
            tnext[ax] = (b.lo[ax] + (idx[ax] + 1) * b.a[ax] - s[ax]) / d[ax];
            tdelta[ax] = b.a[ax] / d[ax];
        } else if (d[ax] < 0.0) {
            step[ax] = -1;
            tnext[ax] = (b.lo[ax] + idx[ax] * b.a[ax] - s[ax]) / d[ax];
            tdelta[ax] = -b.a[ax] / d[ax];
        } else {
            step[ax] = 0;
            tnext[ax] = INFINITY;
            tdelta[ax] = INFINITY;
        }
    }
    double t = t0;
    while (true) {
        const double tn = fmin(tnext[0], fmin(tnext[1], tnext[2]));
        const double len = (fmin(tn, t1) - t) * dlen;
        if (len > 0.0) emit(b.i0[0] + idx[0], b.i0[1] + idx[1], b.i0[2] + idx[2], len);
        if (tn >= t1) return;
        bool left = false;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            if (tnext[ax] == tn) {
                idx[ax] += step[ax];
                if (idx[ax] < 0 || idx[ax] >= b.n[ax]) left = true;
                tnext[ax] += tdelta[ax];
            }
        }
        if (left) return;
        t = tn;
    }
}

__device__ __forceinline__ Box make_box(const Scene& sc, const int* d_box) {
    Box box;
    const double a[3] = {sc.a1, sc.a2, sc.a3};
    const double mn[3] = {sc.minx, sc.miny, sc.minz};
    const int cnt[3] = {sc.n1, sc.n2, sc.n3};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int lo = d_box ? d_box[d] : 0;
        const int hi = d_box ? d_box[3 + d] : cnt[d];
        box.a[d] = a[d];
        box.i0[d] = lo;
        box.n[d] = hi - lo;
        box.lo[d] = mn[d] + lo * a[d];
    }
    return box;
}

template <class T>
__global__ void siddon_fwd_kernel(SiddonLaunch L, const T* __restrict__ vol_in, T* __restrict__ proj_out) {
    const Box box = make_box(L.sc, L.d_box);
    if (box.n[0] <= 0 || box.n[1] <= 0 || box.n[2] <= 0) return;  // all-zero volume
    const int w = L.c1 - L.c0, hgt = L.r1 - L.r0;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= w * hgt) return;
    const int m = L.r0 + idx / w, n = L.c0 + idx % w;
    const int v = L.view_begin + blockIdx.y;
    const ViewConst& vc = L.views[v];
    const double src[3] = {vc.sx, vc.sy, vc.s3};
    const int K = L.k_per_edge;
    const size_t n1 = L.sc.n1, n2 = L.sc.n2;
    double acc = 0.0;
    for (int uu = 0; uu < K; ++uu) {
        const double chi1 = n + (uu + 0.5) / K - 0.5;
        for (int ww = 0; ww < K; ++ww) {
            const double chi2 = m + (ww + 0.5) / K - 0.5;
            double dir[3];
#pragma unroll
            for (int d = 0; d < 3; ++d)
                dir[d] = vc.base[d] + chi1 * vc.du[d] + chi2 * vc.dv[d] - src[d];
            const double dl = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
            traverse(box, src, dir, dl, [&](int i, int j, int k, double chord) {
                acc += double(__ldg(vol_in + (size_t(k) * n2 + j) * n1 + i)) * chord;
            });
        }
    }
    const double inv_k2 = 1.0 / (double(K) * double(K));
    proj_out[size_t(blockIdx.y) * L.sc.rows * L.sc.cols + size_t(m) * L.sc.cols + n] = T(acc * inv_k2);
}

template <class T>
__global__ void siddon_bwd_kernel(SiddonLaunch L, const T* __restrict__ proj_in, T* vol_out) {
    const Box box = make_box(L.sc, nullptr);
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int cols = L.sc.cols, rows = L.sc.rows;
    if (idx >= rows * cols) return;
    const int m = idx / cols, n = idx % cols;
    const int vloc = blockIdx.y;
    const int v = L.view_begin + vloc;
    const int K = L.k_per_edge;
    const double inv_k2 = 1.0 / (double(K) * double(K));
    const double wgt = double(__ldg(proj_in + size_t(vloc) * rows * cols + idx)) * inv_k2;
    if (wgt == 0.0) return;
    const ViewConst& vc = L.views[v];
    const double src[3] = {vc.sx, vc.sy, vc.s3};
    const size_t n1 = L.sc.n1, n2 = L.sc.n2;
    for (int uu = 0; uu < K; ++uu) {
        const double chi1 = n + (uu + 0.5) / K - 0.5;
        for (int ww = 0; ww < K; ++ww) {
            const double chi2 = m + (ww + 0.5) / K - 0.5;
            double dir[3];
#pragma unroll
            for (int d = 0; d < 3; ++d)
                dir[d] = vc.base[d] + chi1 * vc.du[d] + chi2 * vc.dv[d] - src[d];
            const double dl = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
            traverse(box, src, dir, dl, [&](int i, int j, int k, double chord) {
                atomicAdd(vol_out + (size_t(k) * n2 + j) * n1 + i, T(wgt * chord));
            });
        }
    }
}

// Tight box of nonzero voxels (siddon.cpp:182-199): d_box6 = {lo0,lo1,lo2,hi0,hi1,hi2}
// initialised to {N1,N2,N3,0,0,0} by the caller.
template <class T>
__global__ void nonzero_box_kernel(const T* vol, int n1, int n2, int n3, int* box) {
    const size_t total = size_t(n1) * n2 * n3;
    int lo[3] = {n1, n2, n3}, hi[3] = {0, 0, 0};
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        if (vol[idx] != T(0)) {
            const int i = int(idx % n1), j = int((idx / n1) % n2), k = int(idx / (size_t(n1) * n2));
            lo[0] = min(lo[0], i);
            lo[1] = min(lo[1], j);
            lo[2] = min(lo[2], k);
            hi[0] = max(hi[0], i + 1);
            hi[1] = max(hi[1], j + 1);
            hi[2] = max(hi[2], k + 1);
        }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = min(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = max(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    }
    if ((threadIdx.x & 31) == 0) {
        for (int d = 0; d < 3; ++d) {
            atomicMin(box + d, lo[d]);
            atomicMax(box + 3 + d, hi[d]);
        }
    }
}

__global__ void trace_ray_kernel(Scene sc, double sx, double sy, double sz, double tx, double ty,
                                 double tz, int cap, int* ijk, double* len, int* n_out) {
    const Box box = make_box(sc, nullptr);
    const double s[3] = {sx, sy, sz};
    const double d[3] = {tx - sx, ty - sy, tz - sz};
    const double dl = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    int n = 0;
    traverse(box, s, d, dl, [&](int i, int j, int k, double chord) {
        if (n < cap) {
            ijk[3 * n] = i;
            ijk[3 * n + 1] = j;
            ijk[3 * n + 2] = k;
            len[n] = chord;
        }
        ++n;
    });
    *n_out = n;
}

}  // namespace

cudaError_t launch_trace_ray(const Scene& sc, const double* src, const double* tgt, int cap, int* ijk,
                             double* len, int* n_out, cudaStream_t stream) {
    trace_ray_kernel<<<1, 1, 0, stream>>>(sc, src[0], src[1], src[2], tgt[0], tgt[1], tgt[2], cap, ijk,
                                          len, n_out);
    return cudaGetLastError();
}

cudaError_t launch_nonzero_box(const void* vol, bool fp64, const Scene& sc, int* d_box6,
                               cudaStream_t stream) {
    const int init[6] = {sc.n1, sc.n2, sc.n3, 0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(d_box6, init, sizeof(init), cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
    if (fp64)
        nonzero_box_kernel<<<148 * 8, 256, 0, stream>>>(static_cast<const double*>(vol), sc.n1, sc.n2,
                                                        sc.n3, d_box6);
    else
        nonzero_box_kernel<<<148 * 8, 256, 0, stream>>>(static_cast<const float*>(vol), sc.n1, sc.n2,
                                                        sc.n3, d_box6);
    return cudaGetLastError();
}

cudaError_t launch_siddon(const SiddonLaunch& L, bool forward, cudaStream_t stream) {
    if (L.view_count <= 0) return cudaSuccess;
    const Scene& sc = L.sc;
    const size_t esz = L.fp64 ? sizeof(double) : sizeof(float);
    cudaError_t e;
    if (forward) {
        e = cudaMemsetAsync(L.proj_out, 0, esz * size_t(sc.rows) * sc.cols * L.view_count, stream);
        if (e != cudaSuccess) return e;
        const int npx = (L.r1 - L.r0) * (L.c1 - L.c0);
        if (npx <= 0) return cudaSuccess;
        dim3 grid((npx + 127) / 128, L.view_count);
        if (L.fp64)
            siddon_fwd_kernel<double><<<grid, 128, 0, stream>>>(L, static_cast<const double*>(L.vol_in),
                                                                static_cast<double*>(L.proj_out));
        else
            siddon_fwd_kernel<float><<<grid, 128, 0, stream>>>(L, static_cast<const float*>(L.vol_in),
                                                               static_cast<float*>(L.proj_out));
    } else {
        if (!L.accumulate) {
            e = cudaMemsetAsync(L.vol_out, 0, esz * size_t(sc.n1) * sc.n2 * sc.n3, stream);
            if (e != cudaSuccess) return e;
        }
        const int npx = sc.rows * sc.cols;
        dim3 grid((npx + 127) / 128, L.view_count);
        if (L.fp64)
            siddon_bwd_kernel<double><<<grid, 128, 0, stream>>>(L, static_cast<const double*>(L.proj_in),
                                                                static_cast<double*>(L.vol_out));
        else
            siddon_bwd_kernel<float><<<grid, 128, 0, stream>>>(L, static_cast<const float*>(L.proj_in),
                                                               static_cast<float*>(L.vol_out));
    }
    return cudaGetLastError();
}

}  // namespace cvpb
