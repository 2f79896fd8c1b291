// Host-side launch interfaces of the device kernels (internal to libcvpb200).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "common.cuh"

namespace cvpb {

struct CvpLaunch {
    Scene sc;
    const ViewConst* views;   // device, all views of the scene
    const float* scales;      // device, [slots][rows*cols] (mode already selected)
    const float* vol_in;
    float* vol_out;
    const float* proj_in;
    float* proj_out;
    int view_begin, view_count;
    int forward, exact, elevation_correction, cut_centroid;
    int relaxed;              // CvpPrecision::Single (same geometry, see run_cvp)
    int cut_radius_ok = 0;    // relaxed CutCentroid: per-voxel-cut radius kernel (run_cvp)
    int accumulate, deterministic;
    int tile_need;            // largest brick footprint (floats), see launch_cvp_tile_need
    int tall_voxels;          // voxels ~2 detector rows tall: three straight-line rows
    // host-path zero-copy (mapped pinned float64 host buffers, device pointers):
    // forward reads the volume straight from the host while staging bricks;
    // backward writes its (accumulated) result straight to the host
    // scratch for the per-(view, column) cut table (kCutTableBytes per
    // column-view); launches are split into view chunks that fit
    void* cut_table = nullptr;
    size_t cut_table_bytes = 0;
    int cut_table_valid = 0;  // the table already holds views [table_v0, table_v0 + table_nv)
    int table_v0 = 0, table_nv = 0;  // (valid: a superset of this launch's views, same options)
    const double* vol_in64 = nullptr;
    float* vol_copy = nullptr;  // forward with vol_in64: also leave a float32 copy here
    double* vol_out64 = nullptr;
    // forward with ExecPolicy::deterministic: int64 fixed-point merge buffer
    // (view_count x rows x cols) and scratch for its quantum (det_prepare)
    unsigned long long* det_acc = nullptr;
    double* det_g = nullptr;
    unsigned int* det_maxbits = nullptr;
    double det_factor = 0.0;  // voxel count * voxel volume / r_min^2 (bound per unit |mu|)
    // backward: n > 0 adds each brick's result into the owning slab target
    // (float atomics, possibly peer memory) instead of writing vol_out
    SlabTargets targets{};
    int* err;                 // device error flag
};

cudaError_t launch_cvp_tile_need(const Scene& sc, const ViewConst* views, int n_views, int* d_need,
                                 cudaStream_t stream);
cudaError_t launch_cvp(const CvpLaunch& L, cudaStream_t stream);
// the same for brick shape B (cvp_kernels.cu compiled with CVP_CFG_B)
cudaError_t launch_cvp_tile_need_b(const Scene& sc, const ViewConst* views, int n_views, int* d_need,
                                   cudaStream_t stream);
cudaError_t launch_cvp_b(const CvpLaunch& L, cudaStream_t stream);
// and brick shape C (CVP_CFG_C)
cudaError_t launch_cvp_tile_need_c(const Scene& sc, const ViewConst* views, int n_views, int* d_need,
                                   cudaStream_t stream);
cudaError_t launch_cvp_c(const CvpLaunch& L, cudaStream_t stream);
// Only the cut table of views [L.view_begin, L.view_begin + L.view_count)
// (must fit L.cut_table_bytes); later launches over subsets reuse it.
cudaError_t launch_cut_table(const CvpLaunch& L, cudaStream_t stream);
// Per-view work of a launch: the number of voxel-column cuts of views
// [view_begin, view_begin + view_count) in the resident cut table of views
// [table_v0, table_v0 + table_nv), one sum per view into work[0..view_count)
// (zeroed here). view_seconds attributes a launch's time by it.
cudaError_t launch_view_work(void* cut_table, int ncols, int table_v0, int table_nv, int view_begin,
                             int view_count, unsigned long long* work, cudaStream_t stream);
// bytes of cut table per (view, voxel column): count, Q0, rho2c, MAXC x 2 float4
#ifndef CVP_MAXC
#define CVP_MAXC 4
#endif
constexpr int kCutSlots = CVP_MAXC;
constexpr size_t kCutTableBytes = 4 + 8 + 4 + kCutSlots * 32;
cudaError_t launch_scale_image(double f, double pp1, double pp2, double b1, double b2, int rows,
                               int cols, int exact, float* out, double* out64, cudaStream_t stream);
cudaError_t launch_cut_records(const Scene& sc, const ViewConst* views, int view, int i, int j,
                               int k, int exact, int corr, int per_row_r, int clamp, int cap,
                               int* rows, int* cols, double* vol, double* inv, int* n_out, int* err,
                               cudaStream_t stream);

struct SiddonLaunch {
    Scene sc;
    const ViewConst* views;
    // float32 buffers (device API) or float64 (fp64 = 1: the host path)
    const void* vol_in;
    void* vol_out;
    const void* proj_in;
    void* proj_out;
    int fp64;
    int view_begin, view_count;
    int k_per_edge;
    int r0, r1, c0, c1;       // forward ROI (resolved, half-open)
    const int* d_box;         // forward: device {lo0,lo1,lo2,hi0,hi1,hi2} of nonzero voxels
    int accumulate;
};
cudaError_t launch_siddon(const SiddonLaunch& L, bool forward, cudaStream_t stream);
cudaError_t launch_trace_ray(const Scene& sc, const double* src, const double* tgt, int cap, int* ijk,
                             double* len, int* n_out, cudaStream_t stream);
cudaError_t launch_nonzero_box(const void* vol, bool fp64, const Scene& sc, int* d_box6,
                               cudaStream_t stream);

struct TTLaunch {
    Scene sc;
    const ViewConst* views;
    const float* vol_in;
    float* vol_out;
    const float* proj_in;
    float* proj_out;
    int view_begin, view_count;
    int amplitude;
    int accumulate;
};
cudaError_t launch_tt(const TTLaunch& L, bool forward, cudaStream_t stream);

// vector ops (CGLS)
// Device-resident CGLS scalars (cvpb_cgls): status 0 = running, else the
// reference's early exits (solver.cpp:80-105) with the iteration they hit.
enum { kCgFlat = 1, kCgBreakdown = 2, kCgDiverged = 3 };
struct CgState {
    double gamma, alpha, beta;
    int status, iteration;
    int finite;
    int pad;
};
// mode 0: hist[0] = sqrt(sum p1); 1: gamma = sum p1; 2: qq = sum p1 -> alpha;
// 3: gamma_new = sum p1 -> beta, hist[it] = sqrt(sum p2), finite check
cudaError_t launch_cg_scalar(int mode, const double* p1, const double* p2, CgState* st,
                             double* hist, int it, cudaStream_t stream);
cudaError_t launch_cg_update(const CgState* st, float* x, const float* p, size_t n, float* r,
                             const float* q, size_t m, double* partials, int* finite,
                             cudaStream_t stream);
cudaError_t launch_cg_xpby(const CgState* st, const float* s, float* p, size_t n,
                           cudaStream_t stream);
cudaError_t launch_dot(const float* a, const float* b, size_t n, double* d_partials,
                       int n_partials, cudaStream_t stream);
int dot_partials_count();
cudaError_t launch_axpy(double alpha, const float* x, float* y, size_t n, cudaStream_t stream);
cudaError_t launch_xpby(const float* s, double beta, float* p, size_t n, cudaStream_t stream);
cudaError_t launch_all_finite(const float* x, size_t n, int* d_flag, cudaStream_t stream);
cudaError_t launch_sart_residual(const float* b, const float* ax, const float* rowsum, float* out,
                                 size_t n, float eps, cudaStream_t stream);
cudaError_t launch_sart_update(float* x, const float* corr, const float* colsum, float lambda,
                               int nonneg, size_t n, float eps, cudaStream_t stream);
// multi-device exchange (group_kernels.cu): out[i] = sum over members h (fixed
// order, float64) of src.p[h][i] — the z-slab reduce-scatter over peer memory
constexpr int kMaxMembers = 16;
struct SlabSources {
    const float* p[kMaxMembers];
};
cudaError_t launch_reduce_slab(const SlabSources& src, int n, size_t count, float* out,
                               cudaStream_t stream);
cudaError_t launch_reduce_slab64(const SlabSources& src, int n, size_t count, double* out,
                                 cudaStream_t stream);
// error text for the calling thread's cvpb_last_error() (api.cpp)
int set_last_error(int code, const char* msg);
cudaError_t launch_f64_to_f32(const double* in, float* out, size_t n, cudaStream_t stream);
cudaError_t launch_f32_to_f64(const float* in, double* out, size_t n, cudaStream_t stream);

}  // namespace cvpb
