// Shared-memory atomic throughput on one B200 (SURVEY §8d secondary roof:
// "measured B200 shared-memory fp32 atomic throughput ÷ U").
//
// Every CTA hammers its own shared array with conflict-free updates (lane l of
// warp w hits word (w * 32 + l + i * 1024) mod SIZE): one warp-wide
// instruction updates 32 distinct banks. Variants:
//   red.shared.add.s32  (ATOMS.ADD; what the CVP forward's int32 tile uses)
//   red.shared.add.f32  (float add: a CAS loop on sm_100)
//   ld+st.shared.f32    (plain read-modify-write, the backward's gather analogue)
// Reports updates/s over the whole GPU (148 SMs) and per SM clock.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o smem_atomic_peak smem_atomic_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int SIZE = 8192;  // 32 KB of int/float per CTA
constexpr int ITERS = 4096;

template <int MODE>
__global__ void __launch_bounds__(256) hammer(int* out) {
    __shared__ int s[SIZE];
    for (int i = threadIdx.x; i < SIZE; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(s));
    uint32_t idx = threadIdx.x;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        const uint32_t a = base + 4u * ((idx + 1024u * uint32_t(i)) & (SIZE - 1));
        if (MODE == 0) {
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(1) : "memory");
        } else if (MODE == 1) {
            asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(a), "f"(1.0f) : "memory");
        } else {
            float v;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v + 1.0f) : "memory");
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(out, s[0]);
}

template <int MODE>
double run(int blocks, int* d_out, float* ms_out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    hammer<MODE><<<blocks, 256>>>(d_out);  // warm-up
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) hammer<MODE><<<blocks, 256>>>(d_out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms / reps;
    return double(blocks) * 256.0 * ITERS / (ms / reps * 1e-3);
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    int* d_out;
    cudaMalloc(&d_out, sizeof(int));
    const int blocks = sms * 8;  // 8 CTAs x 256 threads per SM (full occupancy at 32 KB smem)
    const char* names[3] = {"red.shared.add.s32", "red.shared.add.f32", "ld+st.shared.f32"};
    printf("{\"sms\": %d, \"sm_clock_mhz_nominal\": %.0f, \"results\": [", sms, clk_khz / 1e3);
    for (int m = 0; m < 3; ++m) {
        float ms = 0.f;
        const double ups = m == 0 ? run<0>(blocks, d_out, &ms) : m == 1 ? run<1>(blocks, d_out, &ms)
                                                                       : run<2>(blocks, d_out, &ms);
        printf("%s{\"op\": \"%s\", \"updates_per_s\": %.4e, \"per_sm_per_nominal_clock\": %.2f, \"ms\": %.3f}",
               m ? ", " : "", names[m], ups, ups / sms / (clk_khz * 1e3), ms);
    }
    printf("]}\n");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
