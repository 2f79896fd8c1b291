// C-ABI of libcvpb200: contexts, scene upload, validation, dispatch to the
// sm_100a kernels, the reference-facing float64 host path and the
// device-resident CGLS driver. See include/cvpb200.h for the contract.
//
// Host geometry follows the reference's semantics (file:line cited per
// function) so that error types, messages and view parameters match; the
// numeric hot path lives in the .cu files.
#include "cvpb200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "kernels.hpp"

using cvpb::Scene;
using cvpb::ViewConst;

namespace {

thread_local std::string g_error;

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

#define CVPB_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(CVPB_CUDA_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                             " at " #call);                                \
    } while (0)

#define CVPB_TRY(call)                 \
    do {                               \
        int rc_ = (call);              \
        if (rc_ != CVPB_OK) return rc_; \
    } while (0)

// ---- tiny float64 vector helpers ------------------------------------------
struct D3 {
    double x, y, z;
};
inline D3 d3(const double* p) { return {p[0], p[1], p[2]}; }
inline double dot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline D3 cross(D3 a, D3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline D3 add(D3 a, D3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline D3 sub(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline D3 mul(double s, D3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double norm(D3 a) { return std::sqrt(dot(a, a)); }

const double kPi = 3.14159265358979323846;

// ---- view validation (ViewGeometry::make, geometry.cpp:52-88) --------------
int view_make(const double s[3], const double fr[9], double f, const double pp[2],
              const double b[2], cvpb_view* out) {
    for (int i = 0; i < 3; ++i)
        if (!std::isfinite(s[i])) return fail(CVPB_INVALID_ARGUMENT, "source is not finite");
    if (!std::isfinite(f)) return fail(CVPB_INVALID_ARGUMENT, "focal length is not finite");
    if (f <= 0.0) return fail(CVPB_INVALID_ARGUMENT, "focal length must be positive");
    if (b[0] <= 0.0 || b[1] <= 0.0) return fail(CVPB_INVALID_ARGUMENT, "pixel sizes must be positive");
    const double tol = 1e-12;
    D3 row[3] = {d3(fr), d3(fr + 3), d3(fr + 6)};
    for (int r = 0; r < 3; ++r)
        for (int c = r; c < 3; ++c) {
            const double want = r == c ? 1.0 : 0.0;
            if (std::abs(dot(row[r], row[c]) - want) > tol)
                return fail(CVPB_INVALID_ARGUMENT, "detector frame is not orthonormal");
        }
    if (std::abs(dot(row[0], cross(row[1], row[2])) - 1.0) > 1e-10)
        return fail(CVPB_INVALID_ARGUMENT, "detector frame must be right-handed");
    if (std::abs(row[1].x) > tol || std::abs(row[1].y) > tol || std::abs(row[1].z + 1.0) > tol)
        return fail(CVPB_INVALID_ARGUMENT, "chi2 axis must be antiparallel to world x3");
    cvpb_view v;
    std::memcpy(v.source, s, sizeof v.source);
    std::memcpy(v.frame, fr, sizeof v.frame);
    v.frame[3] = 0.0;
    v.frame[4] = 0.0;
    v.frame[5] = -1.0;
    v.focal_length = f;
    v.principal_point[0] = pp[0];
    v.principal_point[1] = pp[1];
    v.pixel_size[0] = b[0];
    v.pixel_size[1] = b[1];
    *out = v;
    return CVPB_OK;
}

// Camera rows C = K*Q (geometry.cpp:82-86).
void camera(const cvpb_view& v, D3 cam[3]) {
    const D3 eu = d3(v.frame), ev = d3(v.frame + 3), ew = d3(v.frame + 6);
    const double fu = v.focal_length / v.pixel_size[0], fv = v.focal_length / v.pixel_size[1];
    cam[0] = add(mul(fu, eu), mul(v.principal_point[0], ew));
    cam[1] = add(mul(fv, ev), mul(v.principal_point[1], ew));
    cam[2] = ew;
}

ViewConst view_const(const cvpb_view& v) {
    ViewConst c{};
    D3 cam[3];
    camera(v, cam);
    c.sx = v.source[0];
    c.sy = v.source[1];
    c.s3 = v.source[2];
    c.w1x = cam[0].x;
    c.w1y = cam[0].y;
    c.w3x = cam[2].x;
    c.w3y = cam[2].y;
    c.pp1 = v.principal_point[0];
    c.pp2 = v.principal_point[1];
    c.f_over_b2 = v.focal_length / v.pixel_size[1];
    c.b2_over_f = v.pixel_size[1] / v.focal_length;
    const D3 eu = d3(v.frame), ev = d3(v.frame + 3), ew = d3(v.frame + 6), s = d3(v.source);
    const D3 du = mul(v.pixel_size[0], eu), dv = mul(v.pixel_size[1], ev);
    const D3 base = sub(sub(add(s, mul(v.focal_length, ew)), mul(v.principal_point[0], du)),
                        mul(v.principal_point[1], dv));
    const D3 vecs[6] = {base, du, dv, eu, ev, ew};
    double* dst[6] = {c.base, c.du, c.dv, c.eu, c.ev, c.ew};
    for (int q = 0; q < 6; ++q) {
        dst[q][0] = vecs[q].x;
        dst[q][1] = vecs[q].y;
        dst[q][2] = vecs[q].z;
    }
    c.f = v.focal_length;
    c.b1 = v.pixel_size[0];
    c.b2 = v.pixel_size[1];
    return c;
}

// spherical_quad_area (cvp.cpp:580-599): host API keeps the reference's
// edge-normal form and its domain checks.
int spherical_quad_area(const D3 t[4], double* out) {
    for (int i = 0; i < 4; ++i)
        if (std::abs(norm(t[i]) - 1.0) > 1e-12)
            return fail(CVPB_INVALID_ARGUMENT, "spherical quad vertices must be unit vectors");
    D3 nrm[4];
    for (int i = 0; i < 4; ++i) {
        nrm[i] = cross(t[i], t[(i + 1) % 4]);
        if (dot(nrm[i], nrm[i]) < 1e-30)
            return fail(CVPB_DOMAIN_ERROR, "degenerate spherical quad (parallel consecutive vertices)");
        nrm[i] = mul(1.0 / norm(nrm[i]), nrm[i]);
    }
    double sum = 0.0;
    for (int i = 0; i < 4; ++i)
        sum += std::acos(std::clamp(dot(nrm[i], nrm[(i + 1) % 4]), -1.0, 1.0));
    const double area = 2.0 * kPi - sum;
    if (!(area > 0.0) || !(area < 4.0 * kPi))
        return fail(CVPB_DOMAIN_ERROR, "spherical quad area outside (0, 4*pi)");
    *out = area;
    return CVPB_OK;
}

bool same_intrinsics(const cvpb_view& a, const cvpb_view& b) {
    return a.focal_length == b.focal_length && a.principal_point[0] == b.principal_point[0] &&
           a.principal_point[1] == b.principal_point[1] && a.pixel_size[0] == b.pixel_size[0] &&
           a.pixel_size[1] == b.pixel_size[1];
}

template <class T> struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t reserve(size_t want) {
        if (want <= n && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, sizeof(T) * std::max<size_t>(want, 1));
        if (e == cudaSuccess) n = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

}  // namespace

struct cvpb_context {
    int device = 0;
    cudaStream_t stream = nullptr;  // host-path / CGLS stream
    bool has_geometry = false;
    cvpb_volume_geometry vol{};
    cvpb_detector_geometry det{};
    Scene sc{};
    std::vector<cvpb_view> views;
    std::vector<ViewConst> vconst;
    bool source_inside = false;     // check_view_consistency (cvp.cpp:242-246)
    bool pixel_mismatch = false;    // (cvp.cpp:239-241)
    bool base_reaches_source = false;  // (cvp.cpp:82-84), resolved for the whole box
    int n_slots = 0;
    int cvp_tile_need = 0;    // floats, largest brick footprint over the scene
    int cvp_tile_need_b = 0;  // the same for brick shapes B and C
    int cvp_tile_need_c = 0;
    // brick shape per (direction, precision, elevation, radius): 0 = default,
    // 1 = shape B, 2 = shape C; chosen by timing them on the scene's first launch
    std::map<int, int> cvp_shape;
    double r_min = 0.0;       // smallest source-to-volume-box distance over the views
    double z_far = 0.0;       // largest |z - s3| of the volume box over the views
    double voxel_rows = 0.0;  // mean voxel height in detector rows at the volume centre
    DevBuf<ViewConst> d_views;
    DevBuf<float> d_scale_cos, d_scale_exact;
    DevBuf<int> d_err, d_box, d_flag;
    DevBuf<double> d_partials, d_stage;
    DevBuf<unsigned char> d_cut_table;  // CVP per-(view, column) cut table scratch
    // what the table holds (a single-chunk launch's views and options), and
    // the event after the last launch that read or wrote it: launches on
    // other streams wait for it, so the shared scratch is stream-ordered
    struct {
        int valid = 0, view_begin = 0, view_count = 0, exact = 0, corr = 0;
    } cut_key;
    cudaEvent_t ev_table = nullptr;
    cudaEvent_t ev_tune[2] = {};  // brick-shape timing
    bool ev_table_recorded = false;
    DevBuf<float> h_vol, h_proj;  // device buffers of the host path
    DevBuf<double> h_in64, h_out64;  // float64 host path (Siddon)
    DevBuf<float> cg_r, cg_q, cg_s, cg_p;
    DevBuf<double> cg_partials, cg_hist;
    DevBuf<cvpb::CgState> cg_state;
    DevBuf<unsigned long long> d_det;  // deterministic forward: int64 merge stack
    DevBuf<unsigned long long> d_view_work;  // view_seconds weights (cut counts per view)
    DevBuf<double> d_det_g;
    DevBuf<unsigned int> d_det_max;
    DevBuf<int> d_rec_i;
    DevBuf<double> d_rec_d;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // host path: copy stream + per-chunk events (stack transfers overlap the
    // projector launches of the neighbouring view chunks)
#ifndef CVPB_HOST_CHUNKS
#define CVPB_HOST_CHUNKS 4
#endif
    static constexpr int kChunks = CVPB_HOST_CHUNKS;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_chunk[kChunks] = {};
    cudaEvent_t ev_copy = nullptr;
    size_t nvox() const { return size_t(vol.counts[0]) * vol.counts[1] * vol.counts[2]; }
    size_t npx_view() const { return size_t(det.rows) * det.cols; }
};

namespace {

int check_ctx(cvpb_context* ctx, bool need_geometry = true) {
    if (!ctx) return fail(CVPB_INVALID_ARGUMENT, "null context");
    if (need_geometry && !ctx->has_geometry)
        return fail(CVPB_INVALID_ARGUMENT, "no geometry set on the context");
    if (cudaSetDevice(ctx->device) != cudaSuccess)
        return fail(CVPB_CUDA_ERROR, "cannot select the context's device");
    return CVPB_OK;
}

int check_range(cvpb_context* ctx, int view_begin, int view_count) {
    if (view_begin < 0 || view_count < 0 || view_begin + view_count > int(ctx->views.size()))
        return fail(CVPB_INVALID_ARGUMENT, "projection stack does not match views");
    return CVPB_OK;
}

// check_view_consistency semantics (cvp.cpp:237-247), evaluated per call like
// the reference so the error surfaces from project/backproject.
int check_scene_views(cvpb_context* ctx) {
    if (ctx->pixel_mismatch)
        return fail(CVPB_INVALID_ARGUMENT, "view pixel size does not match the detector geometry");
    if (ctx->source_inside)
        return fail(CVPB_RUNTIME_ERROR, "unsupported configuration: source inside the volume box");
    return CVPB_OK;
}

int check_cvp_options(const cvpb_cvp_options* o) {
    if (!o) return fail(CVPB_INVALID_ARGUMENT, "null CVP options");
    if ((o->scaling != 0 && o->scaling != 1) || (o->precision != 0 && o->precision != 1) ||
        (o->r_estimate != 0 && o->r_estimate != 1))
        return fail(CVPB_INVALID_ARGUMENT, "invalid CVP options");
    return CVPB_OK;
}

int check_siddon_k(int k, const cvpb_exec_policy* exec) {
    if (k < 1) return fail(CVPB_INVALID_ARGUMENT, "Siddon K must be at least 1");
    if (k >= 128 && !(exec && exec->allow_expensive))
        return fail(CVPB_INVALID_ARGUMENT,
                    "Siddon-K with K >= 128 is a deliberately expensive ground-truth "
                    "configuration; set ExecPolicy::allow_expensive to confirm");
    return CVPB_OK;
}

int device_error(cvpb_context* ctx, cudaStream_t st) {
    int h = 0;
    CVPB_CUDA(cudaMemcpyAsync(&h, ctx->d_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CVPB_CUDA(cudaStreamSynchronize(st));
    if (h == 0) return CVPB_OK;
    int zero = 0;
    CVPB_CUDA(cudaMemcpyAsync(ctx->d_err.p, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
    CVPB_CUDA(cudaStreamSynchronize(st));
    if (h & cvpb::kDevSourcePlane)
        return fail(CVPB_RUNTIME_ERROR, "numerical degeneracy: voxel base reaches the source plane");
    return fail(CVPB_DOMAIN_ERROR, "centroid of a degenerate polygon");
}

// Scratch for the CVP cut table of up to `view_count` views: the whole range
// when it fits (c3: 512^2 columns x 496 views = 18.7 GB), else the largest
// view chunk within a third of the free device memory (launch_cvp then splits
// the launch into view chunks).
int reserve_cut_table(cvpb_context* ctx, int view_count, void*& mem, size_t& bytes) {
    const size_t per_view = size_t(ctx->sc.n1) * ctx->sc.n2 * cvpb::kCutTableBytes;
    size_t want = per_view * size_t(std::max(view_count, 1));
    if (ctx->d_cut_table.n < want) {
        size_t free_b = 0, total_b = 0;
        CVPB_CUDA(cudaMemGetInfo(&free_b, &total_b));
        size_t cap = (free_b + ctx->d_cut_table.n) / 3;
        // CVPB_CUT_TABLE_MAX_BYTES caps it further (tests force view chunks)
        if (const char* env = std::getenv("CVPB_CUT_TABLE_MAX_BYTES"))
            cap = std::min(cap, size_t(std::strtoull(env, nullptr, 10)));
        if (want > cap) want = std::max(per_view, cap / per_view * per_view);
        if (ctx->d_cut_table.n < want) {
            // the table's contents go with the old buffer: a later launch
            // must not trust a key that described it
            ctx->cut_key.valid = 0;
            ctx->d_cut_table.release();
            CVPB_CUDA(ctx->d_cut_table.reserve(want));
        }
    }
    mem = ctx->d_cut_table.p;
    bytes = ctx->d_cut_table.n;
    return CVPB_OK;
}

int prepare_cut_table(cvpb_context* ctx, const cvpb_cvp_options* opts, int view_begin,
                      int view_count, cudaStream_t st);

int cvp_tile_need_of(const cvpb_context* ctx, int shape) {
    return shape == 1 ? ctx->cvp_tile_need_b : shape == 2 ? ctx->cvp_tile_need_c : ctx->cvp_tile_need;
}

cudaError_t launch_cvp_shape(const cvpb::CvpLaunch& L, int shape, cudaStream_t st) {
    return shape == 1 ? cvpb::launch_cvp_b(L, st) : shape == 2 ? cvpb::launch_cvp_c(L, st)
                                                               : cvpb::launch_cvp(L, st);
}

int run_cvp(cvpb_context* ctx, const cvpb_cvp_options* opts, const cvpb_exec_policy* exec,
            bool forward, const float* vol_in, float* vol_out, const float* proj_in,
            float* proj_out, int view_begin, int view_count, int accumulate, cudaStream_t st,
            const double* vol_in64 = nullptr, double* vol_out64 = nullptr,
            const cvpb::SlabTargets* targets = nullptr) {
    CVPB_TRY(check_ctx(ctx));
    CVPB_TRY(check_cvp_options(opts));
    CVPB_TRY(check_range(ctx, view_begin, view_count));
    CVPB_TRY(check_scene_views(ctx));
    if (ctx->base_reaches_source)
        return fail(CVPB_RUNTIME_ERROR, "numerical degeneracy: voxel base reaches the source plane");
    cvpb::CvpLaunch L{};
    L.sc = ctx->sc;
    L.views = ctx->d_views.p;
    L.scales = opts->scaling == CVPB_SCALING_EXACT ? ctx->d_scale_exact.p : ctx->d_scale_cos.p;
    L.vol_in = vol_in;
    L.vol_out = vol_out;
    L.proj_in = proj_in;
    L.proj_out = proj_out;
    L.view_begin = view_begin;
    L.view_count = view_count;
    L.forward = forward ? 1 : 0;
    // Both precisions form the world-scale column quantities (depth, chi1,
    // the chi2 anchor) in float64 and run the voxel loop in offset-stable
    // float32: that is what holds the 1e-5 bar for relaxed too (float32
    // world coordinates — the reference's Single semantics — miss it by 6x at
    // c3 on a noise-like stack, tests/test_config_parity_gpu.py).
    L.exact = 1;
    L.relaxed = opts->precision == CVPB_PRECISION_RELAXED ? 1 : 0;
    // relaxed CutCentroid takes one radius per voxel-cut where a brick's
    // bound allows it (kernel footprint()); the variant is only launched for
    // scenes where most bricks qualify (scene bound below; c3 does, the tall
    // configs[3] / [4] volumes do not and keep the per-row kernel)
    {
        const double h = 0.5 * ctx->vol.voxel_size[2];
        L.cut_radius_ok = L.relaxed && ctx->r_min > 0.0 &&
                                  2.0 * (ctx->z_far + h) * h <= 5e-6 * ctx->r_min * ctx->r_min
                              ? 1
                              : 0;
    }
    L.elevation_correction = opts->elevation_correction ? 1 : 0;
    L.cut_centroid = opts->r_estimate == CVPB_R_CUT_CENTROID ? 1 : 0;
    L.accumulate = accumulate;
    L.deterministic = exec ? exec->deterministic : 0;
    L.tile_need = ctx->cvp_tile_need;
    // the three-row straight-line general walk for voxels ~2 rows tall: the
    // forward only (since the three-boundary fast walk took most such bricks,
    // the backward is 3% faster at c2 without its register pressure)
    L.tall_voxels = forward && ctx->voxel_rows > 1.4 ? 1 : 0;
    const void* table_before = ctx->d_cut_table.p;
    CVPB_TRY(reserve_cut_table(ctx, view_count, L.cut_table, L.cut_table_bytes));
    // reuse the resident table when it covers this launch's views with the
    // same options (the P and BP of a step or of one CGLS iteration; the
    // host path's view chunks)
    const size_t per_view = size_t(ctx->sc.n1) * ctx->sc.n2 * cvpb::kCutTableBytes;
    const bool one_chunk = per_view * size_t(view_count) <= L.cut_table_bytes;
    auto& key = ctx->cut_key;
    L.cut_table_valid = key.valid && table_before == L.cut_table && key.view_begin <= view_begin &&
                                view_begin + view_count <= key.view_begin + key.view_count &&
                                key.exact == L.exact && key.corr == L.elevation_correction
                            ? 1
                            : 0;
    L.table_v0 = key.view_begin;
    L.table_nv = key.view_count;
    L.vol_in64 = vol_in64;
    L.vol_copy = vol_in64 ? const_cast<float*>(vol_in) : nullptr;
    L.vol_out64 = vol_out64;
    L.err = ctx->d_err.p;
    if (targets) L.targets = *targets;
    if (forward && L.deterministic && view_count > 0) {
        // bricks merge in int64 fixed point (order-independent): P is
        // bit-reproducible like the reference's deterministic ExecPolicy
        // (exec.hpp:6-15); 8 B per pixel of the launch
        CVPB_CUDA(ctx->d_det.reserve(ctx->npx_view() * size_t(view_count)));
        CVPB_CUDA(ctx->d_det_g.reserve(1));
        CVPB_CUDA(ctx->d_det_max.reserve(1));
        L.det_acc = ctx->d_det.p;
        L.det_g = ctx->d_det_g.p;
        L.det_maxbits = ctx->d_det_max.p;
        const double vv = ctx->vol.voxel_size[0] * ctx->vol.voxel_size[1] * ctx->vol.voxel_size[2];
        L.det_factor = double(ctx->nvox()) * vv / std::max(ctx->r_min * ctx->r_min, 1e-300);
    }
    if (!forward && view_count == 0 && (accumulate || targets)) return CVPB_OK;
    if (!forward && view_count == 0 && !accumulate) {
        CVPB_CUDA(cudaMemsetAsync(vol_out, 0, sizeof(float) * ctx->nvox(), st));
        return CVPB_OK;
    }
    if (!ctx->ev_table) CVPB_CUDA(cudaEventCreateWithFlags(&ctx->ev_table, cudaEventDisableTiming));
    if (ctx->ev_table_recorded) CVPB_CUDA(cudaStreamWaitEvent(st, ctx->ev_table, 0));
    // brick shape: measured once per scene and option set (both shapes on up
    // to 24 of this launch's views, written into this launch's own output,
    // which the real launch then overwrites)
    // (CVPB_CVP_SHAPE=0 / 1 forces a shape, e.g. for tests)
    const int shape_key = (L.forward << 3) | (L.relaxed << 2) | (L.elevation_correction << 1) | L.cut_centroid;
    auto it = ctx->cvp_shape.find(shape_key);
    int shape = it != ctx->cvp_shape.end() ? it->second : 0;
    const char* forced = std::getenv("CVPB_CVP_SHAPE");
    bool tune = false;
    if (forced) {
        shape = std::min(std::max(std::atoi(forced), 0), 2);
    } else if (it == ctx->cvp_shape.end() && view_count >= 8 && (forward || !accumulate) &&
               !vol_in64 && !vol_out64 && !targets) {
        // the timing launches need the whole range's cut table resident
        if (!L.cut_table_valid) {
            CVPB_TRY(prepare_cut_table(ctx, opts, view_begin, view_count, st));
            L.cut_table_valid = key.valid && ctx->d_cut_table.p == L.cut_table ? 1 : 0;
            L.table_v0 = key.view_begin;
            L.table_nv = key.view_count;
        }
        tune = L.cut_table_valid != 0;
    }
    if (tune) {
        cvpb::CvpLaunch T = L;
        T.view_count = std::min(view_count, 24);
        T.accumulate = 0;
        float ms[3] = {0.f, 0.f, 0.f};
        if (!ctx->ev_tune[0])
            for (cudaEvent_t& e : ctx->ev_tune) CVPB_CUDA(cudaEventCreate(&e));
        for (int pass = 0; pass < 2; ++pass)  // pass 0 warms them up
            for (int b = 0; b < 3; ++b) {
                T.tile_need = cvp_tile_need_of(ctx, b);
                CVPB_CUDA(cudaEventRecord(ctx->ev_tune[0], st));
                CVPB_CUDA(launch_cvp_shape(T, b, st));
                CVPB_CUDA(cudaEventRecord(ctx->ev_tune[1], st));
                CVPB_CUDA(cudaEventSynchronize(ctx->ev_tune[1]));
                if (pass) CVPB_CUDA(cudaEventElapsedTime(&ms[b], ctx->ev_tune[0], ctx->ev_tune[1]));
            }
        // another shape only for a clear (> 3%) win over the default
        shape = 0;
        for (int b = 1; b < 3; ++b)
            if (ms[b] < 0.97f * ms[0] && ms[b] < ms[shape]) shape = b;
        ctx->cvp_shape[shape_key] = shape;
    }
    L.tile_need = cvp_tile_need_of(ctx, shape);
    const bool keep = L.cut_table_valid != 0;
    key.valid = 0;
    CVPB_CUDA(launch_cvp_shape(L, shape, st));
    CVPB_CUDA(cudaEventRecord(ctx->ev_table, st));
    ctx->ev_table_recorded = true;
    if (keep) {
        key.valid = 1;  // unchanged
    } else if (one_chunk && view_count > 0) {
        key.valid = 1;
        key.view_begin = view_begin;
        key.view_count = view_count;
        key.exact = L.exact;
        key.corr = L.elevation_correction;
    }
    return CVPB_OK;
}

// Cut table of views [view_begin, view_begin + view_count) ahead of several
// launches over subsets of them (the host path's view chunks); a no-op when
// it does not fit in one piece (the launches then build their own).
int prepare_cut_table(cvpb_context* ctx, const cvpb_cvp_options* opts, int view_begin,
                      int view_count, cudaStream_t st) {
    CVPB_TRY(check_cvp_options(opts));
    CVPB_TRY(check_scene_views(ctx));
    if (ctx->base_reaches_source) return CVPB_OK;  // the launches report it
    cvpb::CvpLaunch L{};
    L.sc = ctx->sc;
    L.views = ctx->d_views.p;
    L.view_begin = view_begin;
    L.view_count = view_count;
    L.exact = 1;  // both precisions: float64 world quantities (see run_cvp)
    L.elevation_correction = opts->elevation_correction ? 1 : 0;
    L.err = ctx->d_err.p;
    auto& key = ctx->cut_key;
    if (key.valid && key.view_begin <= view_begin &&
        view_begin + view_count <= key.view_begin + key.view_count && key.exact == L.exact &&
        key.corr == L.elevation_correction)
        return CVPB_OK;
    CVPB_TRY(reserve_cut_table(ctx, view_count, L.cut_table, L.cut_table_bytes));
    const size_t per_view = size_t(ctx->sc.n1) * ctx->sc.n2 * cvpb::kCutTableBytes;
    if (view_count <= 0 || per_view * size_t(view_count) > L.cut_table_bytes) return CVPB_OK;
    if (!ctx->ev_table) CVPB_CUDA(cudaEventCreateWithFlags(&ctx->ev_table, cudaEventDisableTiming));
    if (ctx->ev_table_recorded) CVPB_CUDA(cudaStreamWaitEvent(st, ctx->ev_table, 0));
    key.valid = 0;
    CVPB_CUDA(cvpb::launch_cut_table(L, st));
    CVPB_CUDA(cudaEventRecord(ctx->ev_table, st));
    ctx->ev_table_recorded = true;
    key.valid = 1;
    key.view_begin = view_begin;
    key.view_count = view_count;
    key.exact = L.exact;
    key.corr = L.elevation_correction;
    return CVPB_OK;
}

int upload_scales(cvpb_context* ctx) {
    // distinct intrinsics -> one scale image per slot (ScaleCache, cvp.cpp:264-302)
    std::vector<int> slot_view;
    for (size_t v = 0; v < ctx->views.size(); ++v) {
        int slot = -1;
        for (size_t s = 0; s < slot_view.size(); ++s)
            if (same_intrinsics(ctx->views[slot_view[s]], ctx->views[v])) {
                slot = int(s);
                break;
            }
        if (slot < 0) {
            slot = int(slot_view.size());
            slot_view.push_back(int(v));
        }
        ctx->vconst[v].scale_slot = slot;
    }
    ctx->n_slots = int(slot_view.size());
    const size_t npx = ctx->npx_view();
    CVPB_CUDA(ctx->d_scale_cos.reserve(npx * ctx->n_slots));
    CVPB_CUDA(ctx->d_scale_exact.reserve(npx * ctx->n_slots));
    for (int s = 0; s < ctx->n_slots; ++s) {
        const cvpb_view& v = ctx->views[slot_view[s]];
        for (int exact = 0; exact < 2; ++exact) {
            float* dst = (exact ? ctx->d_scale_exact.p : ctx->d_scale_cos.p) + npx * s;
            CVPB_CUDA(cvpb::launch_scale_image(v.focal_length, v.principal_point[0],
                                               v.principal_point[1], v.pixel_size[0],
                                               v.pixel_size[1], ctx->det.rows, ctx->det.cols,
                                               exact, dst, nullptr, ctx->stream));
        }
    }
    return CVPB_OK;
}

int ensure_host_buffers(cvpb_context* ctx) {
    const size_t nv = ctx->nvox(), np = ctx->npx_view() * ctx->views.size();
    CVPB_CUDA(ctx->h_vol.reserve(nv));
    CVPB_CUDA(ctx->h_proj.reserve(np));
    CVPB_CUDA(ctx->d_stage.reserve(std::max(nv, np)));
    if (!ctx->copy_stream) {
        CVPB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (cudaEvent_t& e : ctx->ev_chunk) CVPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CVPB_CUDA(cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming));
    }
    return CVPB_OK;
}

// Device pointer of a caller's page-locked (pinned / registered) host buffer,
// or null for pageable memory. The host path reads / writes pinned float64
// volumes in place from the kernels (zero-copy, overlapped with the
// projector) instead of staging them through a bulk copy.
template <class T>
T* mapped_host(T* host) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
    return static_cast<T*>(a.devicePointer);
}

// View chunks of the host path: [begin, end) of chunk c out of n.
int host_chunks(int nviews) { return nviews >= 32 ? cvpb_context::kChunks : 1; }
int chunk_begin(int nviews, int n, int c) { return int((long long)nviews * c / n); }

}  // namespace

namespace {
// H2D(float64 -> float32) of `in`, run(d_in, d_out), D2H(float32 -> float64)
// into `out`; d_in / d_out are the context's host-path device buffers.
template <class Run>
int host_roundtrip(cvpb_context* ctx, bool vol_to_proj, const double* in, double* out, Run&& run) {
    CVPB_TRY(check_ctx(ctx));
    if (!in || !out) return fail(CVPB_INVALID_ARGUMENT, "null host buffer");
    CVPB_TRY(ensure_host_buffers(ctx));
    cudaStream_t st = ctx->stream;
    const size_t nv = ctx->nvox(), np = ctx->npx_view() * ctx->views.size();
    const size_t n_in = vol_to_proj ? nv : np, n_out = vol_to_proj ? np : nv;
    float* d_in = vol_to_proj ? ctx->h_vol.p : ctx->h_proj.p;
    float* d_out = vol_to_proj ? ctx->h_proj.p : ctx->h_vol.p;
    CVPB_CUDA(cudaMemcpyAsync(ctx->d_stage.p, in, sizeof(double) * n_in, cudaMemcpyHostToDevice, st));
    CVPB_CUDA(cvpb::launch_f64_to_f32(ctx->d_stage.p, d_in, n_in, st));
    CVPB_TRY(run(d_in, d_out, st));
    CVPB_CUDA(cvpb::launch_f32_to_f64(d_out, ctx->d_stage.p, n_out, st));
    CVPB_CUDA(cudaMemcpyAsync(out, ctx->d_stage.p, sizeof(double) * n_out, cudaMemcpyDeviceToHost, st));
    CVPB_CUDA(cudaStreamSynchronize(st));
    return CVPB_OK;
}
}  // namespace

namespace cvpb {
int set_last_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace cvpb

extern "C" {

int cvpb_abi_version(void) { return CVPB_ABI_VERSION; }

const char* cvpb_last_error(void) { return g_error.c_str(); }

int cvpb_device_count(int* out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    if (out) *out = n;
    return CVPB_OK;
}

int cvpb_context_create(int device, cvpb_context** out) {
    if (!out) return fail(CVPB_INVALID_ARGUMENT, "null output pointer");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return fail(CVPB_NO_DEVICE, "no CUDA device available (cvpb200 has no CPU fallback)");
    if (device < 0 || device >= n) return fail(CVPB_INVALID_ARGUMENT, "device index out of range");
    CVPB_CUDA(cudaSetDevice(device));
    auto* ctx = new cvpb_context();
    ctx->device = device;
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        ctx->d_err.reserve(1) != cudaSuccess || ctx->d_box.reserve(6) != cudaSuccess ||
        ctx->d_flag.reserve(1) != cudaSuccess ||
        ctx->d_partials.reserve(cvpb::dot_partials_count()) != cudaSuccess ||
        cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) {
        cvpb_context_destroy(ctx);
        return fail(CVPB_CUDA_ERROR, "context allocation failed");
    }
    cudaMemset(ctx->d_err.p, 0, sizeof(int));
    *out = ctx;
    return CVPB_OK;
}

void cvpb_context_destroy(cvpb_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto* b : {&ctx->d_scale_cos, &ctx->d_scale_exact, &ctx->h_vol, &ctx->h_proj, &ctx->cg_r,
                    &ctx->cg_q, &ctx->cg_s, &ctx->cg_p})
        b->release();
    ctx->d_views.release();
    ctx->d_err.release();
    ctx->d_box.release();
    ctx->d_flag.release();
    ctx->d_partials.release();
    ctx->d_stage.release();
    ctx->d_cut_table.release();
    ctx->d_rec_i.release();
    ctx->d_det.release();
    ctx->d_view_work.release();
    ctx->d_det_g.release();
    ctx->d_det_max.release();
    ctx->d_rec_d.release();
    ctx->cg_partials.release();
    ctx->h_in64.release();
    ctx->h_out64.release();
    ctx->cg_hist.release();
    ctx->cg_state.release();
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    for (cudaEvent_t e : ctx->ev_chunk)
        if (e) cudaEventDestroy(e);
    if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
    if (ctx->ev_table) cudaEventDestroy(ctx->ev_table);
    for (cudaEvent_t e : ctx->ev_tune)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int cvpb_set_geometry(cvpb_context* ctx, const cvpb_volume_geometry* vol,
                      const cvpb_detector_geometry* det, int n_views, const cvpb_view* views) {
    CVPB_TRY(check_ctx(ctx, false));
    if (!vol || !det || (n_views > 0 && !views)) return fail(CVPB_INVALID_ARGUMENT, "null geometry");
    // VolumeGeometry::make / DetectorGeometry::make (geometry.cpp:23-50)
    for (int c : vol->counts)
        if (c <= 0) return fail(CVPB_INVALID_ARGUMENT, "voxel counts must be positive");
    for (double a : vol->voxel_size) {
        if (!std::isfinite(a)) return fail(CVPB_INVALID_ARGUMENT, "voxel size is not finite");
        if (a <= 0.0) return fail(CVPB_INVALID_ARGUMENT, "voxel sizes must be positive");
    }
    if (det->rows <= 0 || det->cols <= 0)
        return fail(CVPB_INVALID_ARGUMENT, "detector counts must be positive");
    for (double b : {det->pixel_width, det->pixel_height}) {
        if (!std::isfinite(b)) return fail(CVPB_INVALID_ARGUMENT, "pixel size is not finite");
        if (b <= 0.0) return fail(CVPB_INVALID_ARGUMENT, "pixel sizes must be positive");
    }
    if (n_views < 0) return fail(CVPB_INVALID_ARGUMENT, "negative view count");
    ctx->has_geometry = false;
    ctx->cut_key.valid = 0;
    ctx->vol = *vol;
    ctx->det = *det;
    ctx->views.assign(views, views + n_views);
    for (auto& v : ctx->views) {  // re-validate and snap like ViewGeometry::make
        cvpb_view snapped;
        CVPB_TRY(view_make(v.source, v.frame, v.focal_length, v.principal_point, v.pixel_size,
                           &snapped));
        v = snapped;
    }
    Scene& sc = ctx->sc;
    sc.n1 = vol->counts[0];
    sc.n2 = vol->counts[1];
    sc.n3 = vol->counts[2];
    sc.a1 = vol->voxel_size[0];
    sc.a2 = vol->voxel_size[1];
    sc.a3 = vol->voxel_size[2];
    // min_corner = extent * -0.5 (geometry.hpp:28-29)
    sc.minx = (sc.n1 * sc.a1) * -0.5;
    sc.miny = (sc.n2 * sc.a2) * -0.5;
    sc.minz = (sc.n3 * sc.a3) * -0.5;
    sc.rows = det->rows;
    sc.cols = det->cols;
    sc.pw = det->pixel_width;
    sc.ph = det->pixel_height;
    ctx->vconst.resize(n_views);
    ctx->source_inside = ctx->pixel_mismatch = ctx->base_reaches_source = false;
    const double lo[3] = {sc.minx, sc.miny, sc.minz};
    const double hi[3] = {sc.minx + sc.n1 * sc.a1, sc.miny + sc.n2 * sc.a2, sc.minz + sc.n3 * sc.a3};
    for (int v = 0; v < n_views; ++v) {
        const cvpb_view& vw = ctx->views[v];
        ctx->vconst[v] = view_const(vw);
        if (std::abs(vw.pixel_size[0] - det->pixel_width) > 1e-9 ||
            std::abs(vw.pixel_size[1] - det->pixel_height) > 1e-9)
            ctx->pixel_mismatch = true;
        const double* s = vw.source;
        if (s[0] > lo[0] && s[0] < hi[0] && s[1] > lo[1] && s[1] < hi[1] && s[2] > lo[2] &&
            s[2] < hi[2])
            ctx->source_inside = true;
        double d2 = 0.0;  // squared distance from the source to the box
        for (int q = 0; q < 3; ++q) {
            const double t = std::max(lo[q] - s[q], std::max(0.0, s[q] - hi[q]));
            d2 += t * t;
        }
        ctx->r_min = v == 0 ? std::sqrt(d2) : std::min(ctx->r_min, std::sqrt(d2));
        ctx->z_far = std::max(v == 0 ? 0.0 : ctx->z_far, std::max(std::abs(lo[2] - s[2]), std::abs(hi[2] - s[2])));
        // every voxel-base corner is a convex combination of the box's base
        // corners and depth is affine, so checking the 4 box corners decides
        // the reference's per-voxel depth test (cvp.cpp:82-84) for all voxels
        const ViewConst& c = ctx->vconst[v];
        {
            // voxel height in detector rows at the depth of the volume centre
            const double dc = c.w3x * (0.5 * (lo[0] + hi[0]) - c.sx) + c.w3y * (0.5 * (lo[1] + hi[1]) - c.sy);
            const double rows_v = dc > 0.0 ? sc.a3 * c.f_over_b2 / dc : 0.0;
            ctx->voxel_rows = v == 0 ? rows_v / n_views : ctx->voxel_rows + rows_v / n_views;
        }
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
                const double px = (a ? hi[0] : lo[0]) - c.sx, py = (b ? hi[1] : lo[1]) - c.sy;
                if (!(c.w3x * px + c.w3y * py > 0.0)) ctx->base_reaches_source = true;
            }
    }
    CVPB_CUDA(ctx->d_views.reserve(std::max(n_views, 1)));
    if (n_views > 0)
        CVPB_CUDA(cudaMemcpyAsync(ctx->d_views.p, ctx->vconst.data(), sizeof(ViewConst) * n_views,
                                  cudaMemcpyHostToDevice, ctx->stream));
    CVPB_TRY(upload_scales(ctx));
    if (n_views > 0)  // scale slots were assigned after the first copy
        CVPB_CUDA(cudaMemcpyAsync(ctx->d_views.p, ctx->vconst.data(), sizeof(ViewConst) * n_views,
                                  cudaMemcpyHostToDevice, ctx->stream));
    CVPB_CUDA(cvpb::launch_cvp_tile_need(sc, ctx->d_views.p, n_views, ctx->d_flag.p, ctx->stream));
    CVPB_CUDA(cudaMemcpyAsync(&ctx->cvp_tile_need, ctx->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost,
                              ctx->stream));
    CVPB_CUDA(cudaStreamSynchronize(ctx->stream));
    CVPB_CUDA(cvpb::launch_cvp_tile_need_b(sc, ctx->d_views.p, n_views, ctx->d_flag.p, ctx->stream));
    CVPB_CUDA(cudaMemcpyAsync(&ctx->cvp_tile_need_b, ctx->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost,
                              ctx->stream));
    CVPB_CUDA(cudaStreamSynchronize(ctx->stream));
    CVPB_CUDA(cvpb::launch_cvp_tile_need_c(sc, ctx->d_views.p, n_views, ctx->d_flag.p, ctx->stream));
    CVPB_CUDA(cudaMemcpyAsync(&ctx->cvp_tile_need_c, ctx->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost,
                              ctx->stream));
    CVPB_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->cvp_shape.clear();
    ctx->has_geometry = true;
    return CVPB_OK;
}

int cvpb_get_counts(const cvpb_context* ctx, int* n_views, size_t* volume_elems,
                    size_t* projection_elems) {
    if (!ctx || !ctx->has_geometry) return fail(CVPB_INVALID_ARGUMENT, "no geometry set on the context");
    if (n_views) *n_views = int(ctx->views.size());
    if (volume_elems) *volume_elems = ctx->nvox();
    if (projection_elems) *projection_elems = ctx->npx_view() * ctx->views.size();
    return CVPB_OK;
}

// ---- geometry helpers ------------------------------------------------------

int cvpb_view_make(const double source[3], const double frame[9], double focal_length,
                   const double principal_point[2], const double pixel_size[2], cvpb_view* out) {
    if (!source || !frame || !principal_point || !pixel_size || !out)
        return fail(CVPB_INVALID_ARGUMENT, "null argument");
    return view_make(source, frame, focal_length, principal_point, pixel_size, out);
}

// make_circular_trajectory (geometry.cpp:182-210): source on +x1 at w = 0,
// counter-clockwise; 360 deg arcs are open circles, shorter arcs inclusive.
int cvpb_make_circular_trajectory(double sid, double sdd, int n_views, double arc_deg,
                                  const cvpb_detector_geometry* det, cvpb_view* out) {
    if (!det || !out) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    if (n_views <= 0) return fail(CVPB_INVALID_ARGUMENT, "need at least one view");
    if (!(sid > 0.0) || !(sdd > 0.0)) return fail(CVPB_INVALID_ARGUMENT, "distances must be positive");
    if (!(arc_deg > 0.0) || arc_deg > 360.0)
        return fail(CVPB_INVALID_ARGUMENT, "arc must lie in (0, 360] degrees");
    const double step = std::abs(arc_deg - 360.0) < 1e-9 ? 360.0 / n_views
                                                         : (n_views > 1 ? arc_deg / (n_views - 1) : 0.0);
    const double pp[2] = {(det->cols - 1) * 0.5, (det->rows - 1) * 0.5};
    const double b[2] = {det->pixel_width, det->pixel_height};
    for (int v = 0; v < n_views; ++v) {
        const double w = v * step * kPi / 180.0;
        const double c = std::cos(w), s = std::sin(w);
        const double src[3] = {sid * c, sid * s, 0.0};
        const D3 ew{-c, -s, 0.0}, ev{0.0, 0.0, -1.0};
        const D3 eu = cross(ev, ew);
        const double fr[9] = {eu.x, eu.y, eu.z, ev.x, ev.y, ev.z, ew.x, ew.y, ew.z};
        CVPB_TRY(view_make(src, fr, sdd, pp, b, &out[v]));
    }
    return CVPB_OK;
}

// standard_matrix [C | -C s] (geometry.cpp:120-131).
int cvpb_view_standard_matrix(const cvpb_view* view, double P[12]) {
    if (!view || !P) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    D3 cam[3];
    camera(*view, cam);
    const D3 s = d3(view->source);
    for (int r = 0; r < 3; ++r) {
        P[4 * r + 0] = cam[r].x;
        P[4 * r + 1] = cam[r].y;
        P[4 * r + 2] = cam[r].z;
        P[4 * r + 3] = -dot(cam[r], s);
    }
    return CVPB_OK;
}

// from_standard_matrix (geometry.cpp:133-180): factor P = [B | p4] of any
// scale into source, frame, focal length and principal point.
int cvpb_view_from_standard_matrix(const double P[12], const double pixel_size[2], cvpb_view* out) {
    if (!P || !pixel_size || !out) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    for (int i = 0; i < 12; ++i)
        if (!std::isfinite(P[i])) return fail(CVPB_INVALID_ARGUMENT, "matrix entry is not finite");
    const D3 B0{P[0], P[1], P[2]}, B1{P[4], P[5], P[6]}, B2{P[8], P[9], P[10]};
    const D3 p4{P[3], P[7], P[11]};
    const double detB = dot(B0, cross(B1, B2));
    if (std::abs(detB) < 1e-300) return fail(CVPB_DOMAIN_ERROR, "matrix is singular");
    // B^-1 columns are cross products of row pairs / det
    const D3 c0 = mul(1.0 / detB, cross(B1, B2)), c1 = mul(1.0 / detB, cross(B2, B0)),
             c2 = mul(1.0 / detB, cross(B0, B1));
    const D3 binv_p4{c0.x * p4.x + c1.x * p4.y + c2.x * p4.z, c0.y * p4.x + c1.y * p4.y + c2.y * p4.z,
                     c0.z * p4.x + c1.z * p4.y + c2.z * p4.z};
    const D3 src = mul(-1.0, binv_p4);
    double scl = norm(B2);
    if (!(scl > 0.0)) return fail(CVPB_INVALID_ARGUMENT, "degenerate projection matrix");
    if (detB < 0.0) scl = -scl;
    const D3 C0 = mul(1.0 / scl, B0), C1 = mul(1.0 / scl, B1), C2 = mul(1.0 / scl, B2);
    D3 ew = C2;
    const double pp2 = dot(C1, ew);
    const D3 ev_f = sub(C1, mul(pp2, ew));
    const double fv = norm(ev_f);
    const double pp1 = dot(C0, ew);
    const D3 eu_f = sub(C0, mul(pp1, ew));
    const double fu = norm(eu_f);
    if (!(fu > 0.0) || !(fv > 0.0)) return fail(CVPB_INVALID_ARGUMENT, "degenerate projection matrix");
    const double f = fv * pixel_size[1];
    if (std::abs(fu * pixel_size[0] - f) > 1e-6 * std::abs(f))
        return fail(CVPB_INVALID_ARGUMENT,
                    "projection matrix focal lengths are inconsistent with the pixel sizes");
    const D3 ev = mul(1.0 / fv, ev_f);
    if (std::abs(ev.x) > 1e-6 || std::abs(ev.y) > 1e-6 || std::abs(ev.z + 1.0) > 1e-6)
        return fail(CVPB_INVALID_ARGUMENT, "projection matrix violates the detector row convention");
    const D3 evs{0.0, 0.0, -1.0};
    ew.z = 0.0;
    const double ewn = norm(ew);
    if (!(ewn > 0.0)) return fail(CVPB_DOMAIN_ERROR, "cannot normalize zero vector");
    ew = mul(1.0 / ewn, ew);
    const D3 eu = cross(evs, ew);
    const double s[3] = {src.x, src.y, src.z};
    const double fr[9] = {eu.x, eu.y, eu.z, evs.x, evs.y, evs.z, ew.x, ew.y, ew.z};
    const double pp[2] = {pp1, pp2};
    return view_make(s, fr, f, pp, pixel_size, out);
}

int cvpb_view_project_point(const cvpb_view* view, const double x[3], double chi[2]) {
    if (!view || !x || !chi) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    D3 cam[3];
    camera(*view, cam);
    const D3 d = sub(d3(x), d3(view->source));
    const double w = dot(d3(view->frame + 6), d);
    if (!(w > 0.0))
        return fail(CVPB_DOMAIN_ERROR, "point does not lie strictly on the detector side of the source");
    chi[0] = dot(cam[0], d) / w;
    chi[1] = dot(cam[1], d) / w;
    return CVPB_OK;
}

// pixel_scale_cos / pixel_scale_exact (cvp.cpp:570-605).
int cvpb_pixel_scale(const cvpb_view* view, const cvpb_detector_geometry* det, int exact, int m,
                     int n, double* out) {
    if (!view || !det || !out) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    if (m < 0 || n < 0 || m >= det->rows || n >= det->cols)
        return fail(CVPB_OUT_OF_RANGE, "pixel outside the detector");
    const double f = view->focal_length, pp1 = view->principal_point[0],
                 pp2 = view->principal_point[1], b1 = view->pixel_size[0],
                 b2 = view->pixel_size[1];
    if (!exact) {
        const double u = (n - pp1) * b1, v = (m - pp2) * b2;
        const double c = f / std::sqrt(u * u + v * v + f * f);
        *out = f * f / (det->pixel_width * det->pixel_height * c * c * c);
        return CVPB_OK;
    }
    const double u0 = (n - 0.5 - pp1) * b1, u1 = (n + 0.5 - pp1) * b1;
    const double v0 = (m - 0.5 - pp2) * b2, v1 = (m + 0.5 - pp2) * b2;
    D3 t[4] = {{u0, v0, f}, {u1, v0, f}, {u1, v1, f}, {u0, v1, f}};
    for (auto& q : t) q = mul(1.0 / norm(q), q);
    double omega;
    CVPB_TRY(spherical_quad_area(t, &omega));
    *out = 1.0 / omega;
    return CVPB_OK;
}

int cvpb_fill_uniform01(double* out, size_t n, uint64_t seed) {
    if (!out && n) return fail(CVPB_INVALID_ARGUMENT, "null output");
    std::mt19937_64 rng(seed);
    for (size_t i = 0; i < n; ++i) out[i] = double(rng() >> 11) * 0x1.0p-53;
    return CVPB_OK;
}

// ---- CVP --------------------------------------------------------------------

int cvpb_project_cvp(cvpb_context* ctx, const cvpb_cvp_options* opts, const cvpb_exec_policy* exec,
                     const float* d_volume, float* d_proj, int view_begin, int view_count,
                     void* stream) {
    return run_cvp(ctx, opts, exec, true, d_volume, nullptr, nullptr, d_proj, view_begin,
                   view_count, 0, static_cast<cudaStream_t>(stream));
}

int cvpb_backproject_cvp(cvpb_context* ctx, const cvpb_cvp_options* opts,
                         const cvpb_exec_policy* exec, const float* d_proj, float* d_volume,
                         int view_begin, int view_count, int accumulate, void* stream) {
    return run_cvp(ctx, opts, exec, false, nullptr, d_volume, d_proj, nullptr, view_begin,
                   view_count, accumulate, static_cast<cudaStream_t>(stream));
}

int cvpb_cvp_view_weights(cvpb_context* ctx, const cvpb_cvp_options* opts, int view_begin,
                          int view_count, double* weights) {
    CVPB_TRY(check_ctx(ctx));
    CVPB_TRY(check_cvp_options(opts));
    CVPB_TRY(check_range(ctx, view_begin, view_count));
    if (view_count > 0 && !weights) return fail(CVPB_INVALID_ARGUMENT, "null output");
    if (view_count <= 0) return CVPB_OK;
    cudaStream_t st = ctx->stream;
    CVPB_TRY(prepare_cut_table(ctx, opts, view_begin, view_count, st));
    const auto& key = ctx->cut_key;
    const int corr = opts->elevation_correction ? 1 : 0;
    std::vector<unsigned long long> w(size_t(view_count), 0ull);
    if (key.valid && key.view_begin <= view_begin && view_begin + view_count <= key.view_begin + key.view_count &&
        key.corr == corr) {
        CVPB_CUDA(ctx->d_view_work.reserve(size_t(view_count)));
        if (ctx->ev_table_recorded) CVPB_CUDA(cudaStreamWaitEvent(st, ctx->ev_table, 0));
        CVPB_CUDA(cvpb::launch_view_work(ctx->d_cut_table.p, ctx->sc.n1 * ctx->sc.n2, key.view_begin,
                                         key.view_count, view_begin, view_count, ctx->d_view_work.p, st));
        CVPB_CUDA(cudaEventRecord(ctx->ev_table, st));
        ctx->ev_table_recorded = true;
        CVPB_CUDA(cudaMemcpyAsync(w.data(), ctx->d_view_work.p, sizeof(unsigned long long) * view_count,
                                  cudaMemcpyDeviceToHost, st));
        CVPB_CUDA(cudaStreamSynchronize(st));
    }
    // (a range whose table does not fit in one piece: equal weights)
    double sum = 0.0;
    for (unsigned long long x : w) sum += double(x);
    for (int v = 0; v < view_count; ++v) weights[v] = sum > 0.0 ? double(w[v]) / sum : 1.0 / view_count;
    return CVPB_OK;
}

namespace {
// view_seconds of a host call: the call's measured time (ev0 .. ev1)
// attributed to the views by cvpb_cvp_view_weights.
int fill_view_seconds(cvpb_context* ctx, const cvpb_cvp_options* opts, int nviews, double* view_seconds) {
    float ms = 0.f;
    CVPB_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    CVPB_TRY(cvpb_cvp_view_weights(ctx, opts, 0, nviews, view_seconds));
    for (int v = 0; v < nviews; ++v) view_seconds[v] *= ms * 1e-3;
    return CVPB_OK;
}
}  // namespace

int cvpb_ipc_alloc(cvpb_context* ctx, size_t bytes, void** d_ptr, unsigned char handle[64]) {
    CVPB_TRY(check_ctx(ctx, false));
    if (!d_ptr || !handle) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
    void* p = nullptr;
    CVPB_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 1)));
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        CVPB_CUDA(e);
    }
    std::memcpy(handle, &h, 64);
    *d_ptr = p;
    return CVPB_OK;
}

int cvpb_ipc_open(cvpb_context* ctx, const unsigned char handle[64], void** d_ptr) {
    CVPB_TRY(check_ctx(ctx, false));
    if (!d_ptr || !handle) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    CVPB_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return CVPB_OK;
}

int cvpb_ipc_close(cvpb_context* ctx, void* d_ptr) {
    CVPB_TRY(check_ctx(ctx, false));
    if (d_ptr) CVPB_CUDA(cudaIpcCloseMemHandle(d_ptr));
    return CVPB_OK;
}

int cvpb_ipc_free(cvpb_context* ctx, void* d_ptr) {
    CVPB_TRY(check_ctx(ctx, false));
    if (d_ptr) CVPB_CUDA(cudaFree(d_ptr));
    return CVPB_OK;
}

int cvpb_sync(cvpb_context* ctx, void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    CVPB_CUDA(cudaStreamSynchronize(st));
    return device_error(ctx, st);
}

int cvpb_backproject_cvp_scatter(cvpb_context* ctx, const cvpb_cvp_options* opts,
                                 const cvpb_exec_policy* exec, const float* d_proj, int view_begin,
                                 int view_count, const cvpb_slab_targets* targets, void* stream) {
    CVPB_TRY(check_ctx(ctx));
    if (!targets) return fail(CVPB_INVALID_ARGUMENT, "null slab targets");
    if (exec && exec->deterministic && !targets->store)
        return fail(CVPB_INVALID_ARGUMENT,
                    "atomic slab targets are not bit-reproducible "
                    "(store = 1 + cvpb_sum_slabs for ExecPolicy::deterministic)");
    const int n = targets->n;
    if (n < 1 || n > cvpb::kMaxSlabTargets)
        return fail(CVPB_INVALID_ARGUMENT, "slab targets: 1 to 16 slabs");
    const int n3 = ctx->vol.counts[2];
    if (targets->plane_begin[0] != 0 || targets->plane_begin[n] != n3)
        return fail(CVPB_INVALID_ARGUMENT, "slab targets must cover the volume's planes [0, N3)");
    cvpb::SlabTargets tg;
    tg.n = n;
    for (int t = 0; t <= n; ++t) {
        if (t > 0 && targets->plane_begin[t] < targets->plane_begin[t - 1])
            return fail(CVPB_INVALID_ARGUMENT, "slab target planes must not decrease");
        tg.plane_begin[t] = targets->plane_begin[t];
    }
    for (int t = 0; t < n; ++t) {
        if (!targets->slab[t] && targets->plane_begin[t + 1] > targets->plane_begin[t])
            return fail(CVPB_INVALID_ARGUMENT, "null slab target");
        tg.slab[t] = targets->slab[t];
    }
    tg.store = targets->store ? 1 : 0;
    if (!d_proj && view_count > 0) return fail(CVPB_INVALID_ARGUMENT, "null projection buffer");
    if (view_count == 0 && tg.store) {
        // nothing to backproject: store mode still overwrites with zeros
        for (int t = 0; t < n; ++t) {
            const size_t cnt = size_t(tg.plane_begin[t + 1] - tg.plane_begin[t]) * ctx->sc.n1 * ctx->sc.n2;
            if (cnt) CVPB_CUDA(cudaMemsetAsync(tg.slab[t], 0, sizeof(float) * cnt, static_cast<cudaStream_t>(stream)));
        }
        return CVPB_OK;
    }
    return run_cvp(ctx, opts, exec, false, nullptr, nullptr, d_proj, nullptr, view_begin, view_count,
                   tg.store ? 0 : 1, static_cast<cudaStream_t>(stream), nullptr, nullptr, &tg);
}

int cvpb_sum_slabs(cvpb_context* ctx, const float* const* src, int n, size_t count, float* out32,
                   double* out64, void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    if (n < 1 || n > cvpb::kMaxMembers) return fail(CVPB_INVALID_ARGUMENT, "1 to 16 slabs");
    if (!src || (!out32 && !out64) || (out32 && out64))
        return fail(CVPB_INVALID_ARGUMENT, "sum_slabs: sources and exactly one output");
    cvpb::SlabSources ss{};
    for (int h = 0; h < n; ++h) {
        if (!src[h] && count) return fail(CVPB_INVALID_ARGUMENT, "null slab source");
        ss.p[h] = src[h];
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (out32) CVPB_CUDA(cvpb::launch_reduce_slab(ss, n, count, out32, st));
    else CVPB_CUDA(cvpb::launch_reduce_slab64(ss, n, count, out64, st));
    return CVPB_OK;
}

int cvpb_project_cvp_host(cvpb_context* ctx, const cvpb_cvp_options* opts,
                          const cvpb_exec_policy* exec, const double* volume, double* proj,
                          double* view_seconds) {
    CVPB_TRY(check_ctx(ctx));
    if (!volume || !proj) return fail(CVPB_INVALID_ARGUMENT, "null host buffer");
    CVPB_TRY(ensure_host_buffers(ctx));
    cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
    const size_t nv = ctx->nvox(), npx = ctx->npx_view();
    const int nviews = int(ctx->views.size());
    // this call reports its own device errors only
    CVPB_CUDA(cudaMemsetAsync(ctx->d_err.p, 0, sizeof(int), st));
    CVPB_CUDA(cudaEventRecord(ctx->ev0, st));
    // pinned input: the first chunk's bricks read it in place and leave a
    // float32 device copy for the later chunks (pageable input: one bulk
    // copy first)
    const double* vol_map = mapped_host(volume);
    if (!vol_map) {
        CVPB_CUDA(cudaMemcpyAsync(ctx->d_stage.p, volume, sizeof(double) * nv, cudaMemcpyHostToDevice, st));
        CVPB_CUDA(cvpb::launch_f64_to_f32(ctx->d_stage.p, ctx->h_vol.p, nv, st));
    }
    // view chunks: chunk c's projections go back to the host (float64) on the
    // copy stream while chunk c + 1 is projected; one cut table serves them all
    const int n = host_chunks(nviews);
    if (n > 1) CVPB_TRY(prepare_cut_table(ctx, opts, 0, nviews, st));
    for (int c = 0; c < n; ++c) {
        const int v0 = chunk_begin(nviews, n, c), v1 = chunk_begin(nviews, n, c + 1);
        const size_t off = npx * size_t(v0), cnt = npx * size_t(v1 - v0);
        CVPB_TRY(run_cvp(ctx, opts, exec, true, ctx->h_vol.p, nullptr, nullptr, ctx->h_proj.p + off,
                         v0, v1 - v0, 0, st, c == 0 ? vol_map : nullptr));
        CVPB_CUDA(cudaEventRecord(ctx->ev_chunk[c], st));
        CVPB_CUDA(cudaStreamWaitEvent(cs, ctx->ev_chunk[c], 0));
        CVPB_CUDA(cvpb::launch_f32_to_f64(ctx->h_proj.p + off, ctx->d_stage.p + off, cnt, cs));
        CVPB_CUDA(cudaMemcpyAsync(proj + off, ctx->d_stage.p + off, sizeof(double) * cnt,
                                  cudaMemcpyDeviceToHost, cs));
    }
    CVPB_CUDA(cudaEventRecord(ctx->ev_copy, cs));
    CVPB_CUDA(cudaStreamWaitEvent(st, ctx->ev_copy, 0));
    CVPB_CUDA(cudaEventRecord(ctx->ev1, st));
    CVPB_TRY(device_error(ctx, st));
    if (view_seconds) CVPB_TRY(fill_view_seconds(ctx, opts, nviews, view_seconds));
    return CVPB_OK;
}

int cvpb_backproject_cvp_host(cvpb_context* ctx, const cvpb_cvp_options* opts,
                              const cvpb_exec_policy* exec, const double* proj, double* volume,
                              double* view_seconds) {
    CVPB_TRY(check_ctx(ctx));
    if (!volume || !proj) return fail(CVPB_INVALID_ARGUMENT, "null host buffer");
    CVPB_TRY(ensure_host_buffers(ctx));
    cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
    const size_t nv = ctx->nvox(), npx = ctx->npx_view();
    const int nviews = int(ctx->views.size());
    CVPB_CUDA(cudaMemsetAsync(ctx->d_err.p, 0, sizeof(int), st));
    CVPB_CUDA(cudaEventRecord(ctx->ev0, st));
    CVPB_CUDA(cudaStreamWaitEvent(cs, ctx->ev0, 0));
    // view chunks: chunk c + 1 of the stack comes in (float64 -> float32) on
    // the copy stream while chunk c is backprojected; chunks accumulate
    const int n = host_chunks(nviews);
    for (int c = 0; c < n; ++c) {
        const int v0 = chunk_begin(nviews, n, c), v1 = chunk_begin(nviews, n, c + 1);
        const size_t off = npx * size_t(v0), cnt = npx * size_t(v1 - v0);
        CVPB_CUDA(cudaMemcpyAsync(ctx->d_stage.p + off, proj + off, sizeof(double) * cnt,
                                  cudaMemcpyHostToDevice, cs));
        CVPB_CUDA(cvpb::launch_f64_to_f32(ctx->d_stage.p + off, ctx->h_proj.p + off, cnt, cs));
        CVPB_CUDA(cudaEventRecord(ctx->ev_chunk[c], cs));
    }
    // pinned output: the last chunk's bricks write the float64 result in place
    double* vol_map = mapped_host(volume);
    if (n > 1) CVPB_TRY(prepare_cut_table(ctx, opts, 0, nviews, st));
    for (int c = 0; c < n; ++c) {
        const int v0 = chunk_begin(nviews, n, c), v1 = chunk_begin(nviews, n, c + 1);
        CVPB_CUDA(cudaStreamWaitEvent(st, ctx->ev_chunk[c], 0));
        CVPB_TRY(run_cvp(ctx, opts, exec, false, nullptr, ctx->h_vol.p,
                         ctx->h_proj.p + npx * size_t(v0), nullptr, v0, v1 - v0, c > 0 ? 1 : 0, st,
                         nullptr, c == n - 1 ? vol_map : nullptr));
    }
    if (!vol_map) {
        CVPB_CUDA(cvpb::launch_f32_to_f64(ctx->h_vol.p, ctx->d_stage.p, nv, st));
        CVPB_CUDA(cudaMemcpyAsync(volume, ctx->d_stage.p, sizeof(double) * nv, cudaMemcpyDeviceToHost, st));
    }
    CVPB_CUDA(cudaEventRecord(ctx->ev1, st));
    CVPB_TRY(device_error(ctx, st));
    if (view_seconds) CVPB_TRY(fill_view_seconds(ctx, opts, nviews, view_seconds));
    return CVPB_OK;
}

// The host path's backward with the result left in device memory: float64
// host stack in (view chunks H2D + converted on the copy stream, overlapped
// with the bricks of the previous chunk), float32 partial volume out on the
// caller's stream — what a view-sharded rank hands to its cross-device
// reduce-scatter (bench.py N > 1, parallel.py).
int cvpb_backproject_cvp_host_partial(cvpb_context* ctx, const cvpb_cvp_options* opts,
                                      const cvpb_exec_policy* exec, const double* proj,
                                      float* d_volume, void* stream) {
    CVPB_TRY(check_ctx(ctx));
    if (!proj || !d_volume) return fail(CVPB_INVALID_ARGUMENT, "null buffer");
    CVPB_TRY(ensure_host_buffers(ctx));
    cudaStream_t st = static_cast<cudaStream_t>(stream), cs = ctx->copy_stream;
    const size_t npx = ctx->npx_view();
    const int nviews = int(ctx->views.size());
    CVPB_CUDA(cudaEventRecord(ctx->ev0, st));
    CVPB_CUDA(cudaStreamWaitEvent(cs, ctx->ev0, 0));
    const int n = host_chunks(nviews);
    for (int c = 0; c < n; ++c) {
        const int v0 = chunk_begin(nviews, n, c), v1 = chunk_begin(nviews, n, c + 1);
        const size_t off = npx * size_t(v0), cnt = npx * size_t(v1 - v0);
        CVPB_CUDA(cudaMemcpyAsync(ctx->d_stage.p + off, proj + off, sizeof(double) * cnt,
                                  cudaMemcpyHostToDevice, cs));
        CVPB_CUDA(cvpb::launch_f64_to_f32(ctx->d_stage.p + off, ctx->h_proj.p + off, cnt, cs));
        CVPB_CUDA(cudaEventRecord(ctx->ev_chunk[c], cs));
    }
    if (n > 1) CVPB_TRY(prepare_cut_table(ctx, opts, 0, nviews, st));
    for (int c = 0; c < n; ++c) {
        const int v0 = chunk_begin(nviews, n, c), v1 = chunk_begin(nviews, n, c + 1);
        CVPB_CUDA(cudaStreamWaitEvent(st, ctx->ev_chunk[c], 0));
        CVPB_TRY(run_cvp(ctx, opts, exec, false, nullptr, d_volume, ctx->h_proj.p + npx * size_t(v0),
                         nullptr, v0, v1 - v0, c > 0 ? 1 : 0, st));
    }
    if (nviews == 0) CVPB_CUDA(cudaMemsetAsync(d_volume, 0, sizeof(float) * ctx->nvox(), st));
    return CVPB_OK;
}

// float32 device vector -> float64 host buffer (pinned: written in place by
// the conversion kernel; pageable: staged), synchronous.
int cvpb_vec_to_host64(cvpb_context* ctx, const float* d_in, double* host, size_t n, void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    if ((!d_in || !host) && n) return fail(CVPB_INVALID_ARGUMENT, "null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (double* mapped = mapped_host(host)) {
        CVPB_CUDA(cvpb::launch_f32_to_f64(d_in, mapped, n, st));
    } else {
        CVPB_CUDA(ctx->d_stage.reserve(std::max(ctx->d_stage.n, n)));
        CVPB_CUDA(cvpb::launch_f32_to_f64(d_in, ctx->d_stage.p, n, st));
        CVPB_CUDA(cudaMemcpyAsync(host, ctx->d_stage.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    }
    CVPB_CUDA(cudaStreamSynchronize(st));
    return CVPB_OK;
}

int cvpb_collect_cut_records(cvpb_context* ctx, const cvpb_cvp_options* opts, int view, int i,
                             int j, int k, int clamp, int cap, int* rows, int* cols,
                             double* volume, double* inv_r2, int* n_out) {
    CVPB_TRY(check_ctx(ctx));
    CVPB_TRY(check_cvp_options(opts));
    if (view < 0 || view >= int(ctx->views.size()))
        return fail(CVPB_OUT_OF_RANGE, "view index outside the scene");
    if (i < 0 || j < 0 || k < 0 || i >= ctx->sc.n1 || j >= ctx->sc.n2 || k >= ctx->sc.n3)
        return fail(CVPB_OUT_OF_RANGE, "voxel index outside lattice");
    CVPB_TRY(check_scene_views(ctx));
    if (cap < 0) cap = 0;
    cudaStream_t st = ctx->stream;
    CVPB_CUDA(cudaMemsetAsync(ctx->d_err.p, 0, sizeof(int), st));
    CVPB_CUDA(ctx->d_rec_i.reserve(2 * size_t(cap) + 1));
    CVPB_CUDA(ctx->d_rec_d.reserve(2 * size_t(cap) + 1));
    int* d_rows = ctx->d_rec_i.p;
    int* d_cols = d_rows + cap;
    int* d_n = d_cols + cap;
    double* d_vol = ctx->d_rec_d.p;
    double* d_inv = d_vol + cap;
    CVPB_CUDA(cvpb::launch_cut_records(ctx->sc, ctx->d_views.p, view, i, j, k,
                                       1,  // float64 world quantities in both precisions
                                       opts->elevation_correction,
                                       opts->r_estimate == CVPB_R_CUT_CENTROID, clamp, cap, d_rows,
                                       d_cols, d_vol, d_inv, d_n, ctx->d_err.p, st));
    int n = 0;
    CVPB_CUDA(cudaMemcpyAsync(&n, d_n, sizeof(int), cudaMemcpyDeviceToHost, st));
    CVPB_TRY(device_error(ctx, st));
    const int c = std::min(n, cap);
    if (c > 0) {
        if (rows) CVPB_CUDA(cudaMemcpy(rows, d_rows, sizeof(int) * c, cudaMemcpyDeviceToHost));
        if (cols) CVPB_CUDA(cudaMemcpy(cols, d_cols, sizeof(int) * c, cudaMemcpyDeviceToHost));
        if (volume) CVPB_CUDA(cudaMemcpy(volume, d_vol, sizeof(double) * c, cudaMemcpyDeviceToHost));
        if (inv_r2) CVPB_CUDA(cudaMemcpy(inv_r2, d_inv, sizeof(double) * c, cudaMemcpyDeviceToHost));
    }
    if (n_out) *n_out = n;
    return CVPB_OK;
}

int cvpb_scale_image(cvpb_context* ctx, int view, int exact, double* out_host) {
    CVPB_TRY(check_ctx(ctx));
    if (view < 0 || view >= int(ctx->views.size()))
        return fail(CVPB_OUT_OF_RANGE, "view index outside the scene");
    if (!out_host) return fail(CVPB_INVALID_ARGUMENT, "null output");
    const size_t npx = ctx->npx_view();
    DevBuf<double> tmp;
    CVPB_CUDA(tmp.reserve(npx));
    const cvpb_view& v = ctx->views[view];
    cudaError_t e = cvpb::launch_scale_image(v.focal_length, v.principal_point[0],
                                             v.principal_point[1], v.pixel_size[0], v.pixel_size[1],
                                             ctx->det.rows, ctx->det.cols, exact, nullptr, tmp.p,
                                             ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpy(out_host, tmp.p, sizeof(double) * npx, cudaMemcpyDeviceToHost);
    tmp.release();
    CVPB_CUDA(e);
    return CVPB_OK;
}

// ---- Siddon-K -----------------------------------------------------------------

}  // extern "C"

namespace {
// Siddon-K launches over float32 (device API) or float64 (host path) buffers.
int siddon_project(cvpb_context* ctx, int k_per_edge, const cvpb_pixel_roi* roi,
                   const cvpb_exec_policy* exec, const void* d_volume, void* d_proj, int view_begin,
                   int view_count, bool fp64, cudaStream_t st) {
    CVPB_TRY(check_ctx(ctx));
    CVPB_TRY(check_siddon_k(k_per_edge, exec));
    CVPB_TRY(check_range(ctx, view_begin, view_count));
    CVPB_TRY(check_scene_views(ctx));
    cvpb::SiddonLaunch L{};
    L.sc = ctx->sc;
    L.views = ctx->d_views.p;
    L.vol_in = d_volume;
    L.proj_out = d_proj;
    L.fp64 = fp64 ? 1 : 0;
    L.view_begin = view_begin;
    L.view_count = view_count;
    L.k_per_edge = k_per_edge;
    // resolve (siddon.cpp:125-132)
    const int R = ctx->sc.rows, Cc = ctx->sc.cols;
    cvpb_pixel_roi r = roi ? *roi : cvpb_pixel_roi{0, -1, 0, -1};
    L.r0 = std::clamp(r.row_begin, 0, R);
    L.r1 = r.row_end < 0 ? R : std::clamp(r.row_end, L.r0, R);
    L.c0 = std::clamp(r.col_begin, 0, Cc);
    L.c1 = r.col_end < 0 ? Cc : std::clamp(r.col_end, L.c0, Cc);
    CVPB_CUDA(cvpb::launch_nonzero_box(d_volume, fp64, ctx->sc, ctx->d_box.p, st));
    L.d_box = ctx->d_box.p;
    CVPB_CUDA(cvpb::launch_siddon(L, true, st));
    return CVPB_OK;
}

int siddon_backproject(cvpb_context* ctx, int k_per_edge, const cvpb_exec_policy* exec,
                       const void* d_proj, void* d_volume, int view_begin, int view_count,
                       int accumulate, bool fp64, cudaStream_t st) {
    CVPB_TRY(check_ctx(ctx));
    CVPB_TRY(check_siddon_k(k_per_edge, exec));
    CVPB_TRY(check_range(ctx, view_begin, view_count));
    CVPB_TRY(check_scene_views(ctx));
    cvpb::SiddonLaunch L{};
    L.sc = ctx->sc;
    L.views = ctx->d_views.p;
    L.proj_in = d_proj;
    L.vol_out = d_volume;
    L.fp64 = fp64 ? 1 : 0;
    L.view_begin = view_begin;
    L.view_count = view_count;
    L.k_per_edge = k_per_edge;
    L.accumulate = accumulate;
    if (view_count == 0 && !accumulate) {
        CVPB_CUDA(cudaMemsetAsync(d_volume, 0, (fp64 ? sizeof(double) : sizeof(float)) * ctx->nvox(), st));
        return CVPB_OK;
    }
    CVPB_CUDA(cvpb::launch_siddon(L, false, st));
    return CVPB_OK;
}

// Host path of the float64 projectors: H2D of the float64 input, the kernels
// on float64 device buffers, D2H of the float64 output (no conversions).
template <class Run>
int host_roundtrip64(cvpb_context* ctx, bool vol_to_proj, const double* in, double* out, Run&& run) {
    CVPB_TRY(check_ctx(ctx));
    if (!in || !out) return fail(CVPB_INVALID_ARGUMENT, "null host buffer");
    cudaStream_t st = ctx->stream;
    const size_t nv = ctx->nvox(), np = ctx->npx_view() * ctx->views.size();
    const size_t n_in = vol_to_proj ? nv : np, n_out = vol_to_proj ? np : nv;
    CVPB_CUDA(ctx->h_in64.reserve(n_in));
    CVPB_CUDA(ctx->h_out64.reserve(n_out));
    CVPB_CUDA(cudaMemcpyAsync(ctx->h_in64.p, in, sizeof(double) * n_in, cudaMemcpyHostToDevice, st));
    CVPB_TRY(run(ctx->h_in64.p, ctx->h_out64.p, st));
    CVPB_CUDA(cudaMemcpyAsync(out, ctx->h_out64.p, sizeof(double) * n_out, cudaMemcpyDeviceToHost, st));
    CVPB_CUDA(cudaStreamSynchronize(st));
    return CVPB_OK;
}
}  // namespace

extern "C" {

int cvpb_project_siddon(cvpb_context* ctx, int k_per_edge, const cvpb_pixel_roi* roi,
                        const cvpb_exec_policy* exec, const float* d_volume, float* d_proj,
                        int view_begin, int view_count, void* stream) {
    return siddon_project(ctx, k_per_edge, roi, exec, d_volume, d_proj, view_begin, view_count, false,
                          static_cast<cudaStream_t>(stream));
}

int cvpb_backproject_siddon(cvpb_context* ctx, int k_per_edge, const cvpb_exec_policy* exec,
                            const float* d_proj, float* d_volume, int view_begin, int view_count,
                            int accumulate, void* stream) {
    return siddon_backproject(ctx, k_per_edge, exec, d_proj, d_volume, view_begin, view_count,
                              accumulate, false, static_cast<cudaStream_t>(stream));
}

int cvpb_trace_ray(cvpb_context* ctx, const cvpb_volume_geometry* vol, const double source[3],
                   const double target[3], int cap, int* ijk, double* length, int* n_out) {
    CVPB_TRY(check_ctx(ctx, false));
    if (!vol || !source || !target || !n_out) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    for (int c : vol->counts)
        if (c <= 0) return fail(CVPB_INVALID_ARGUMENT, "voxel counts must be positive");
    const double d[3] = {target[0] - source[0], target[1] - source[1], target[2] - source[2]};
    if (!(d[0] * d[0] + d[1] * d[1] + d[2] * d[2] > 0.0))
        return fail(CVPB_INVALID_ARGUMENT, "ray source and target coincide");
    Scene sc{};
    sc.n1 = vol->counts[0];
    sc.n2 = vol->counts[1];
    sc.n3 = vol->counts[2];
    sc.a1 = vol->voxel_size[0];
    sc.a2 = vol->voxel_size[1];
    sc.a3 = vol->voxel_size[2];
    sc.minx = (sc.n1 * sc.a1) * -0.5;
    sc.miny = (sc.n2 * sc.a2) * -0.5;
    sc.minz = (sc.n3 * sc.a3) * -0.5;
    // require_source_outside (siddon.cpp:100-105)
    const double lo[3] = {sc.minx, sc.miny, sc.minz};
    const double hi[3] = {-sc.minx, -sc.miny, -sc.minz};
    if (source[0] > lo[0] && source[0] < hi[0] && source[1] > lo[1] && source[1] < hi[1] &&
        source[2] > lo[2] && source[2] < hi[2])
        return fail(CVPB_RUNTIME_ERROR, "unsupported configuration: source inside the volume box");
    if (cap < 0) cap = 0;
    cudaStream_t st = ctx->stream;
    CVPB_CUDA(ctx->d_rec_i.reserve(3 * size_t(cap) + 1));
    CVPB_CUDA(ctx->d_rec_d.reserve(size_t(cap) + 1));
    int* d_n = ctx->d_rec_i.p + 3 * size_t(cap);
    CVPB_CUDA(cvpb::launch_trace_ray(sc, source, target, cap, ctx->d_rec_i.p, ctx->d_rec_d.p, d_n, st));
    int n = 0;
    CVPB_CUDA(cudaMemcpyAsync(&n, d_n, sizeof(int), cudaMemcpyDeviceToHost, st));
    CVPB_CUDA(cudaStreamSynchronize(st));
    const int c = std::min(n, cap);
    if (c > 0) {
        if (ijk) CVPB_CUDA(cudaMemcpy(ijk, ctx->d_rec_i.p, sizeof(int) * 3 * c, cudaMemcpyDeviceToHost));
        if (length) CVPB_CUDA(cudaMemcpy(length, ctx->d_rec_d.p, sizeof(double) * c, cudaMemcpyDeviceToHost));
    }
    *n_out = n;
    return CVPB_OK;
}

// ---- TT -------------------------------------------------------------------------

int cvpb_project_tt(cvpb_context* ctx, const cvpb_tt_options* opts, const float* d_volume,
                    float* d_proj, int view_begin, int view_count, void* stream) {
    CVPB_TRY(check_ctx(ctx));
    CVPB_TRY(check_range(ctx, view_begin, view_count));
    CVPB_TRY(check_scene_views(ctx));
    cvpb::TTLaunch L{};
    L.sc = ctx->sc;
    L.views = ctx->d_views.p;
    L.vol_in = d_volume;
    L.proj_out = d_proj;
    L.view_begin = view_begin;
    L.view_count = view_count;
    L.amplitude = opts ? opts->amplitude : 1;
    CVPB_CUDA(cvpb::launch_tt(L, true, static_cast<cudaStream_t>(stream)));
    return CVPB_OK;
}

int cvpb_backproject_tt(cvpb_context* ctx, const cvpb_tt_options* opts, const float* d_proj,
                        float* d_volume, int view_begin, int view_count, int accumulate,
                        void* stream) {
    CVPB_TRY(check_ctx(ctx));
    CVPB_TRY(check_range(ctx, view_begin, view_count));
    CVPB_TRY(check_scene_views(ctx));
    cvpb::TTLaunch L{};
    L.sc = ctx->sc;
    L.views = ctx->d_views.p;
    L.proj_in = d_proj;
    L.vol_out = d_volume;
    L.view_begin = view_begin;
    L.view_count = view_count;
    L.amplitude = opts ? opts->amplitude : 1;
    L.accumulate = accumulate;
    CVPB_CUDA(cvpb::launch_tt(L, false, static_cast<cudaStream_t>(stream)));
    return CVPB_OK;
}

// ---- host paths for Siddon-K / TT / CGLS ---------------------------------------


// Siddon's host path runs in float64 end to end, like the reference (it is
// the ground-truth projector: Siddon512 in acceptance.cpp:100-147).
int cvpb_project_siddon_host(cvpb_context* ctx, int k_per_edge, const cvpb_pixel_roi* roi,
                             const cvpb_exec_policy* exec, const double* volume, double* proj) {
    const int V = ctx ? int(ctx->views.size()) : 0;
    return host_roundtrip64(ctx, true, volume, proj, [&](double* din, double* dout, cudaStream_t st) {
        return siddon_project(ctx, k_per_edge, roi, exec, din, dout, 0, V, true, st);
    });
}

int cvpb_backproject_siddon_host(cvpb_context* ctx, int k_per_edge, const cvpb_exec_policy* exec,
                                 const double* proj, double* volume) {
    const int V = ctx ? int(ctx->views.size()) : 0;
    return host_roundtrip64(ctx, false, proj, volume, [&](double* din, double* dout, cudaStream_t st) {
        return siddon_backproject(ctx, k_per_edge, exec, din, dout, 0, V, 0, true, st);
    });
}

int cvpb_project_tt_host(cvpb_context* ctx, const cvpb_tt_options* opts, const double* volume,
                         double* proj) {
    const int V = ctx ? int(ctx->views.size()) : 0;
    return host_roundtrip(ctx, true, volume, proj, [&](float* din, float* dout, cudaStream_t st) {
        return cvpb_project_tt(ctx, opts, din, dout, 0, V, st);
    });
}

int cvpb_backproject_tt_host(cvpb_context* ctx, const cvpb_tt_options* opts, const double* proj,
                             double* volume) {
    const int V = ctx ? int(ctx->views.size()) : 0;
    return host_roundtrip(ctx, false, proj, volume, [&](float* din, float* dout, cudaStream_t st) {
        return cvpb_backproject_tt(ctx, opts, din, dout, 0, V, 0, st);
    });
}

int cvpb_cgls_host(cvpb_context* ctx, int projector, const cvpb_cvp_options* cvp_opts,
                   const cvpb_tt_options* tt_opts, const cvpb_exec_policy* exec, int k_per_edge,
                   const double* b, double* x, int iterations, double* residual_norms) {
    return host_roundtrip(ctx, false, b, x, [&](float* din, float* dout, cudaStream_t st) {
        return cvpb_cgls(ctx, projector, cvp_opts, tt_opts, exec, k_per_edge, din, dout,
                         iterations, residual_norms, st);
    });
}

// ---- vector ops -------------------------------------------------------------------

int cvpb_vec_dot(cvpb_context* ctx, const float* a, const float* b, size_t n, double* out_host,
                 void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    if (!out_host) return fail(CVPB_INVALID_ARGUMENT, "null output");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int np = cvpb::dot_partials_count();
    CVPB_CUDA(cvpb::launch_dot(a, b, n, ctx->d_partials.p, np, st));
    std::vector<double> h(np);
    CVPB_CUDA(cudaMemcpyAsync(h.data(), ctx->d_partials.p, sizeof(double) * np,
                              cudaMemcpyDeviceToHost, st));
    CVPB_CUDA(cudaStreamSynchronize(st));
    double sum = 0.0, c = 0.0;
    for (double x : h) {
        const double y = x - c;
        const double t = sum + y;
        c = (t - sum) - y;
        sum = t;
    }
    *out_host = sum;
    return CVPB_OK;
}

int cvpb_vec_axpy(cvpb_context* ctx, double alpha, const float* x, float* y, size_t n, void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    CVPB_CUDA(cvpb::launch_axpy(alpha, x, y, n, static_cast<cudaStream_t>(stream)));
    return CVPB_OK;
}

int cvpb_vec_xpby(cvpb_context* ctx, const float* s, double beta, float* p, size_t n, void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    CVPB_CUDA(cvpb::launch_xpby(s, beta, p, n, static_cast<cudaStream_t>(stream)));
    return CVPB_OK;
}

int cvpb_vec_all_finite(cvpb_context* ctx, const float* x, size_t n, int* out_host, void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    if (!out_host) return fail(CVPB_INVALID_ARGUMENT, "null output");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int one = 1;
    CVPB_CUDA(cudaMemcpyAsync(ctx->d_flag.p, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    CVPB_CUDA(cvpb::launch_all_finite(x, n, ctx->d_flag.p, st));
    int h = 1;
    CVPB_CUDA(cudaMemcpyAsync(&h, ctx->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CVPB_CUDA(cudaStreamSynchronize(st));
    *out_host = h;
    return CVPB_OK;
}

int cvpb_vec_sart_residual(cvpb_context* ctx, const float* b, const float* ax, const float* rowsum,
                           float* out, size_t n, void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    CVPB_CUDA(cvpb::launch_sart_residual(b, ax, rowsum, out, n, 1e-30f,
                                         static_cast<cudaStream_t>(stream)));
    return CVPB_OK;
}

int cvpb_vec_sart_update(cvpb_context* ctx, float* x, const float* corr, const float* colsum,
                         double lambda, int nonneg, size_t n, void* stream) {
    CVPB_TRY(check_ctx(ctx, false));
    CVPB_CUDA(cvpb::launch_sart_update(x, corr, colsum, float(lambda), nonneg, n, 1e-30f,
                                       static_cast<cudaStream_t>(stream)));
    return CVPB_OK;
}

// ---- device-resident CGLS (solver.cpp:55-106) ------------------------------------
// Per iteration: A p -> q, q.q partials, alpha (device scalar kernel), one
// fused pass x += alpha p / r -= alpha q / r.r partials / finite check,
// A^T r -> s, s.s partials, beta + history entry (device), p = s + beta p.
// gamma, alpha and beta never leave the device; the host reads the 4-word
// status once per iteration (the reference's early exits need it).

int cvpb_cgls(cvpb_context* ctx, int projector, const cvpb_cvp_options* cvp_opts,
              const cvpb_tt_options* tt_opts, const cvpb_exec_policy* exec, int k_per_edge,
              const float* d_b, float* d_x, int iterations, double* residual_norms, void* stream) {
    CVPB_TRY(check_ctx(ctx));
    if (iterations < 1) return fail(CVPB_INVALID_ARGUMENT, "cgls needs at least one iteration");
    if (!d_b || !d_x || !residual_norms) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    if (projector < 0 || projector > 2) return fail(CVPB_INVALID_ARGUMENT, "unknown projector");
    cvpb_cvp_options defaults{CVPB_SCALING_EXACT, 1, CVPB_PRECISION_EXACT, CVPB_R_CUT_CENTROID};
    const cvpb_cvp_options* opts = cvp_opts ? cvp_opts : &defaults;
    CVPB_TRY(check_cvp_options(opts));
    const cvpb_exec_policy ex = exec ? *exec : cvpb_exec_policy{0, 0, 0};
    if (projector == 1) CVPB_TRY(check_siddon_k(k_per_edge, &ex));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t n = ctx->nvox(), m = ctx->npx_view() * ctx->views.size();
    const int V = int(ctx->views.size());
    const int np = cvpb::dot_partials_count();
    CVPB_CUDA(ctx->cg_r.reserve(m));
    CVPB_CUDA(ctx->cg_q.reserve(m));
    CVPB_CUDA(ctx->cg_s.reserve(n));
    CVPB_CUDA(ctx->cg_p.reserve(n));
    CVPB_CUDA(ctx->cg_partials.reserve(2 * size_t(np)));
    CVPB_CUDA(ctx->cg_hist.reserve(size_t(iterations) + 1));
    CVPB_CUDA(ctx->cg_state.reserve(1));
    float *r = ctx->cg_r.p, *q = ctx->cg_q.p, *s = ctx->cg_s.p, *p = ctx->cg_p.p;
    double *pa = ctx->cg_partials.p, *pb = pa + np, *hist = ctx->cg_hist.p;
    cvpb::CgState* state = ctx->cg_state.p;
    auto forward = [&](const float* x, float* out) -> int {
        if (projector == 0) return cvpb_project_cvp(ctx, opts, &ex, x, out, 0, V, st);
        if (projector == 1) return cvpb_project_siddon(ctx, k_per_edge, nullptr, &ex, x, out, 0, V, st);
        return cvpb_project_tt(ctx, tt_opts, x, out, 0, V, st);
    };
    auto adjoint = [&](const float* b, float* out) -> int {
        if (projector == 0) return cvpb_backproject_cvp(ctx, opts, &ex, b, out, 0, V, 0, st);
        if (projector == 1) return cvpb_backproject_siddon(ctx, k_per_edge, &ex, b, out, 0, V, 0, st);
        return cvpb_backproject_tt(ctx, tt_opts, b, out, 0, V, 0, st);
    };
    CVPB_CUDA(cudaMemcpyAsync(r, d_b, sizeof(float) * m, cudaMemcpyDeviceToDevice, st));
    CVPB_CUDA(cudaMemsetAsync(d_x, 0, sizeof(float) * n, st));
    CVPB_CUDA(cudaMemsetAsync(state, 0, sizeof(cvpb::CgState), st));
    CVPB_CUDA(cvpb::launch_dot(r, r, m, pa, np, st));
    CVPB_CUDA(cvpb::launch_cg_scalar(0, pa, pb, state, hist, 0, st));
    CVPB_TRY(adjoint(r, s));
    CVPB_CUDA(cudaMemcpyAsync(p, s, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
    CVPB_CUDA(cvpb::launch_dot(s, s, n, pa, np, st));
    CVPB_CUDA(cvpb::launch_cg_scalar(1, pa, pb, state, hist, 0, st));
    cvpb::CgState h{};
    int done = 0;  // iterations whose history entry is final on the device
    for (int it = 1; it <= iterations; ++it) {
        CVPB_TRY(forward(p, q));
        CVPB_CUDA(cvpb::launch_dot(q, q, m, pa, np, st));
        CVPB_CUDA(cvpb::launch_cg_scalar(2, pa, pb, state, hist, it, st));
        CVPB_CUDA(cvpb::launch_cg_update(state, d_x, p, n, r, q, m, pb, &state->finite, st));
        CVPB_TRY(adjoint(r, s));
        CVPB_CUDA(cvpb::launch_dot(s, s, n, pa, np, st));
        CVPB_CUDA(cvpb::launch_cg_scalar(3, pa, pb, state, hist, it, st));
        CVPB_CUDA(cvpb::launch_cg_xpby(state, s, p, n, st));
        CVPB_CUDA(cudaMemcpyAsync(&h, state, sizeof h, cudaMemcpyDeviceToHost, st));
        CVPB_CUDA(cudaStreamSynchronize(st));
        done = it;
        if (h.status != 0) break;
    }
    CVPB_CUDA(cudaMemcpyAsync(residual_norms, hist, sizeof(double) * (done + 1),
                              cudaMemcpyDeviceToHost, st));
    CVPB_CUDA(cudaStreamSynchronize(st));
    if (h.status == cvpb::kCgBreakdown)
        return fail(CVPB_RUNTIME_ERROR,
                    "CGLS breakdown (A p = 0) at iteration " + std::to_string(h.iteration));
    if (h.status == cvpb::kCgDiverged)
        return fail(CVPB_RUNTIME_ERROR,
                    "CGLS diverged (non-finite iterate) at iteration " + std::to_string(h.iteration));
    for (int it = done + 1; it <= iterations; ++it)  // gamma == 0: the history stays flat
        residual_norms[it] = residual_norms[it - 1];
    return CVPB_OK;
}

}  // extern "C"
