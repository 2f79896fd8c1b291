// Cross-device exchange kernels of the multi-device scene (group.cpp).
//
// The backprojection's exchange step ("BP sums per-GPU partial
// volumes with a reduce-scatter over z-slabs") is one kernel per member that
// reads the z-slab it owns straight out of every member's partial volume over
// NVLink peer memory (UVA loads; the group enables peer access at creation)
// and writes the sum — no NCCL staging copies, no intermediate buffers. The
// members are summed in a fixed order in float64, so the result does not
// depend on timing, and rounds once to the output type: float32 for the
// device-resident CGLS slab, float64 for the host path (the reference's
// AttenuationVolume is float64).
#include <algorithm>
#include <cstdint>

#include "kernels.hpp"

namespace cvpb {

namespace {

template <class Out>
__device__ __forceinline__ void store4(Out* p, double a, double b, double c, double d);

template <>
__device__ __forceinline__ void store4<float>(float* p, double a, double b, double c, double d) {
    *reinterpret_cast<float4*>(p) = make_float4(float(a), float(b), float(c), float(d));
}

template <>
__device__ __forceinline__ void store4<double>(double* p, double a, double b, double c, double d) {
    reinterpret_cast<double2*>(p)[0] = make_double2(a, b);
    reinterpret_cast<double2*>(p)[1] = make_double2(c, d);
}

// out[i] = sum_h src.p[h][i], h = 0..n-1 in order, i < count. VEC: every
// source and the output are 16-byte aligned (float4 loads, 4 outputs per
// thread); the tail (count % 4) is scalar.
template <class Out, bool VEC>
__global__ void __launch_bounds__(256) reduce_slab_kernel(SlabSources src, int n, size_t count,
                                                          Out* __restrict__ out) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    const size_t tid = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    size_t done = 0;
    if (VEC) {
        const size_t n4 = count / 4;
        for (size_t i = tid; i < n4; i += stride) {
            double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
            for (int h = 0; h < n; ++h) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(src.p[h]) + i);
                a += v.x;
                b += v.y;
                c += v.z;
                d += v.w;
            }
            store4<Out>(out + 4 * i, a, b, c, d);
        }
        done = n4 * 4;
    }
    for (size_t i = done + tid; i < count; i += stride) {
        double a = 0.0;
        for (int h = 0; h < n; ++h) a += __ldg(src.p[h] + i);
        out[i] = Out(a);
    }
}

template <class Out>
cudaError_t launch_reduce(const SlabSources& src, int n, size_t count, Out* out, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    bool vec = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    for (int h = 0; h < n; ++h) vec = vec && (reinterpret_cast<uintptr_t>(src.p[h]) & 15u) == 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t work = vec ? (count + 3) / 4 : count;
    const int blocks = int(std::min<size_t>((work + 255) / 256, size_t(sms) * 8));
    if (vec)
        reduce_slab_kernel<Out, true><<<blocks, 256, 0, st>>>(src, n, count, out);
    else
        reduce_slab_kernel<Out, false><<<blocks, 256, 0, st>>>(src, n, count, out);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_reduce_slab(const SlabSources& src, int n, size_t count, float* out,
                               cudaStream_t stream) {
    return launch_reduce<float>(src, n, count, out, stream);
}

cudaError_t launch_reduce_slab64(const SlabSources& src, int n, size_t count, double* out,
                                 cudaStream_t stream) {
    return launch_reduce<double>(src, n, count, out, stream);
}

}  // namespace cvpb
