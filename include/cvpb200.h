/* cvpb200 — B200-native cone-beam projector pair (CVP exact/relaxed, Siddon-K,
 * TT footprint) behind a plain C ABI.
 *
 * This is the drop-in boundary for the reference's C++ operator API
 * (/root/reference/proj/include/cbct/{geometry,cvp,siddon,solver}.hpp). Every
 * entry point cites the reference interface it replaces. No torch or CUDA types
 * cross this boundary: device buffers are raw pointers, streams are opaque
 * `void*` (a cudaStream_t; NULL = the legacy default stream).
 *
 * Data layout (identical to the reference so callers need no reshuffle):
 *   volume     float32[N3][N2][N1]        (i fastest, k slowest; geometry.hpp:34-36)
 *   projection float32[V][rows][cols]     (view-major, rows top->bottom; volume.hpp:23-46)
 * The *_host entry points take the reference's float64 host buffers instead.
 *
 * Errors: every call returns a cvpb_status. The code maps 1:1 onto the
 * exception type the reference throws for the same condition; the message is
 * available from cvpb_last_error() (thread-local).
 */
#ifndef CVPB200_H
#define CVPB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVPB_ABI_VERSION 3

typedef enum cvpb_status {
    CVPB_OK = 0,
    CVPB_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    CVPB_RUNTIME_ERROR = 2,    /* std::runtime_error */
    CVPB_OUT_OF_RANGE = 3,     /* std::out_of_range */
    CVPB_DOMAIN_ERROR = 4,     /* std::domain_error */
    CVPB_CUDA_ERROR = 5,       /* device failure (reported as std::runtime_error) */
    CVPB_NO_DEVICE = 6         /* no CUDA device: the path has no CPU fallback */
} cvpb_status;

/* VolumeGeometry (geometry.hpp:15-39): N1 x N2 x N3 voxels of a1 x a2 x a3 mm,
 * box centred at the world origin. */
typedef struct cvpb_volume_geometry {
    int counts[3];
    double voxel_size[3];
} cvpb_volume_geometry;

/* DetectorGeometry (geometry.hpp:43-56). */
typedef struct cvpb_detector_geometry {
    int rows;
    int cols;
    double pixel_width;  /* b1, along chi1 (columns) */
    double pixel_height; /* b2, along chi2 (rows) */
} cvpb_detector_geometry;

/* ViewGeometry (geometry.hpp:70-123): source, frame rows (e_u, e_v, e_w),
 * focal length f, principal point (pixels), pixel size (mm). 17 doubles. */
typedef struct cvpb_view {
    double source[3];
    double frame[9];
    double focal_length;
    double principal_point[2];
    double pixel_size[2];
} cvpb_view;

/* CvpOptions (cvp.hpp:13-22); enum values follow the reference's declaration
 * order. Defaults: {CVPB_SCALING_EXACT, 1, CVPB_PRECISION_EXACT, CVPB_R_CUT_CENTROID}. */
enum { CVPB_SCALING_COS = 0, CVPB_SCALING_EXACT = 1 };
enum { CVPB_PRECISION_EXACT = 0 /* CvpPrecision::Double */, CVPB_PRECISION_RELAXED = 1 /* ::Single */ };
enum { CVPB_R_VOXEL_CENTER = 0, CVPB_R_CUT_CENTROID = 1 };
typedef struct cvpb_cvp_options {
    int scaling;
    int elevation_correction;
    int precision;
    int r_estimate;
} cvpb_cvp_options;

/* ExecPolicy (exec.hpp:6-15). threads is ignored on the device. deterministic
 * keeps one view group per brick in the CVP backprojection (fixed accumulation
 * order: bit-reproducible); the CVP forward always sums a brick's records in
 * int32 fixed point (order-independent) and merges bricks with float atomics
 * (reproducible to float32 reassociation). allow_expensive gates Siddon
 * K >= 128 exactly as the reference does (siddon.cpp:107-113). */
typedef struct cvpb_exec_policy {
    int threads;
    int deterministic;
    int allow_expensive;
} cvpb_exec_policy;

/* PixelRoi (siddon.hpp:28-33): half-open ranges, end < 0 = full extent. */
typedef struct cvpb_pixel_roi {
    int row_begin;
    int row_end;
    int col_begin;
    int col_end;
} cvpb_pixel_roi;

/* TT footprint options (no reference symbol: SPEC.md:8 leaves TT out; the
 * build defines it after Long, Fessler & Balter 2010, SF-TT with the A2
 * amplitude). */
typedef struct cvpb_tt_options {
    int amplitude; /* 0 = A1 (ray through voxel centre), 1 = A2 (per-pixel ray) */
} cvpb_tt_options;

typedef struct cvpb_context cvpb_context;

/* ---- library / context -------------------------------------------------- */
int cvpb_abi_version(void);
const char* cvpb_last_error(void);
/* The device-buffer calls are asynchronous: geometry degeneracies a kernel
 * detects (voxel base reaching the source plane -> CVPB_RUNTIME_ERROR, a
 * degenerate cut polygon -> CVPB_DOMAIN_ERROR, the reference's exceptions)
 * are raised as device flags. cvpb_sync waits for `stream` (NULL: the
 * context's own stream) and reports and clears the flags raised since the
 * last report; the host-buffer calls do this themselves. */
int cvpb_sync(cvpb_context* ctx, void* stream);
int cvpb_device_count(int* out);
int cvpb_context_create(int device, cvpb_context** out);
void cvpb_context_destroy(cvpb_context* ctx);

/* Upload one scene. Replaces the reference's per-call view list
 * (std::span<const ViewGeometry>, cvp.hpp:87-99) with a resident one: per-view
 * constants (camera rows, source, 1/f ...) are precomputed in float64 on the
 * host and kept in device memory; pixel-scale images are built once per
 * distinct intrinsics (ScaleCache, cvp.cpp:264-302). Validates every view like
 * check_view_consistency (cvp.cpp:237-247). */
int cvpb_set_geometry(cvpb_context* ctx, const cvpb_volume_geometry* vol,
                      const cvpb_detector_geometry* det, int n_views, const cvpb_view* views);
int cvpb_get_counts(const cvpb_context* ctx, int* n_views, size_t* volume_elems,
                    size_t* projection_elems);

/* ---- geometry helpers (geometry.cpp) ------------------------------------ */
/* ViewGeometry::make (geometry.cpp:52-88): validates and snaps the frame. */
int cvpb_view_make(const double source[3], const double frame[9], double focal_length,
                   const double principal_point[2], const double pixel_size[2], cvpb_view* out);
/* make_circular_trajectory (geometry.cpp:182-210). */
int cvpb_make_circular_trajectory(double sid, double sdd, int n_views, double arc_deg,
                                  const cvpb_detector_geometry* det, cvpb_view* out);
/* ViewGeometry::standard_matrix / from_standard_matrix (geometry.cpp:120-180). */
int cvpb_view_standard_matrix(const cvpb_view* view, double P[12]);
int cvpb_view_from_standard_matrix(const double P[12], const double pixel_size[2], cvpb_view* out);
/* ViewGeometry::project_point (geometry.cpp:90-96). */
int cvpb_view_project_point(const cvpb_view* view, const double x[3], double chi[2]);
/* pixel_scale_cos / pixel_scale_exact (cvp.cpp:570-605), host float64. */
int cvpb_pixel_scale(const cvpb_view* view, const cvpb_detector_geometry* det, int exact, int m,
                     int n, double* out);
/* fill_uniform01 (solver.cpp:30-33): mt19937_64, (x >> 11) * 2^-53. */
int cvpb_fill_uniform01(double* out, size_t n, uint64_t seed);

/* ---- CVP (cvp.hpp:81-99) — device buffers ------------------------------- */
/* Every CVP call first computes the column cuts of its views into a device
 * cut table owned by the context (144 B per voxel column and view; at most a
 * third of the free device memory, further capped by the environment variable
 * CVPB_CUT_TABLE_MAX_BYTES; larger jobs run in view chunks). The table stays
 * allocated until the context is destroyed.
 * The first launch per option set with >= 8 views also times the three brick
 * shapes of the kernels on up to 24 of its views (into its own output) and
 * synchronizes the stream once to read the timings; CVPB_CVP_SHAPE=0|1|2
 * skips that (e.g. before capturing a CUDA graph). */
/* project_cvp_into (cvp.cpp:615-626): overwrites views [view_begin,
 * view_begin+view_count) of d_proj (which points at view 0's image of that
 * range, i.e. the caller's slice). */
int cvpb_project_cvp(cvpb_context* ctx, const cvpb_cvp_options* opts,
                     const cvpb_exec_policy* exec, const float* d_volume, float* d_proj,
                     int view_begin, int view_count, void* stream);
/* backproject_cvp_into (cvp.cpp:636-650): accumulate = 0 zero-fills d_volume
 * first (reference semantics, cvp.cpp:645); 1 adds (view-chunked / per-rank
 * partial volumes). */
int cvpb_backproject_cvp(cvpb_context* ctx, const cvpb_cvp_options* opts,
                         const cvpb_exec_policy* exec, const float* d_proj, float* d_volume,
                         int view_begin, int view_count, int accumulate, void* stream);

/* Backprojection fused with the reduce-scatter of a view-sharded job (SURVEY
 * §8e): each brick's voxels go straight into the buffer that owns their
 * z-plane — typically another GPU's memory, reached over NVLink peer access —
 * as soon as the brick has walked its views, so the exchange overlaps the
 * bricks still computing and no partial volume is materialized. Planes
 * [plane_begin[t], plane_begin[t+1]) go to slab[t] (its element 0 is the
 * first voxel of plane plane_begin[t]); plane_begin[0] = 0, plane_begin[n] =
 * N3. The caller orders the slabs against this stream.
 *   store = 1: the launch's result OVERWRITES the regions (plain stores; a
 *     rank writes its own receive region of each owner, and the owner sums
 *     its regions in a fixed order with cvpb_sum_slabs: deterministic);
 *   store = 0: the result is ADDED with float atomics into regions the
 *     caller zeroed (atomic order varies: ExecPolicy::deterministic refused). */
typedef struct cvpb_slab_targets {
    int n; /* 1..16 */
    int plane_begin[17];
    float* slab[16];
    int store;
} cvpb_slab_targets;
/* out[i] = sum over h = 0..n-1, in that order, of src[h][i] (float64
 * accumulation), into out32 (float32) or out64 (float64) — the owner's half
 * of the reduce-scatter above. n <= 16. Asynchronous on `stream`. */
int cvpb_sum_slabs(cvpb_context* ctx, const float* const* src, int n, size_t count, float* out32,
                   double* out64, void* stream);
int cvpb_backproject_cvp_scatter(cvpb_context* ctx, const cvpb_cvp_options* opts,
                                 const cvpb_exec_policy* exec, const float* d_proj, int view_begin,
                                 int view_count, const cvpb_slab_targets* targets, void* stream);

/* Device buffers shared between processes (CUDA IPC), so one process per GPU
 * can run cvpb_backproject_cvp_scatter into the other ranks' slabs: alloc
 * exports a 64-byte handle of a fresh buffer on the context's device; open
 * maps another process's buffer (peer access enabled on demand); close
 * unmaps it; free releases an allocated buffer. */
int cvpb_ipc_alloc(cvpb_context* ctx, size_t bytes, void** d_ptr, unsigned char handle[64]);
int cvpb_ipc_open(cvpb_context* ctx, const unsigned char handle[64], void** d_ptr);
int cvpb_ipc_close(cvpb_context* ctx, void* d_ptr);
int cvpb_ipc_free(cvpb_context* ctx, void* d_ptr);

/* ---- CVP — reference-facing host path (float64 host buffers, H2D/D2H inside) */
int cvpb_project_cvp_host(cvpb_context* ctx, const cvpb_cvp_options* opts,
                          const cvpb_exec_policy* exec, const double* volume, double* proj,
                          double* view_seconds);
int cvpb_backproject_cvp_host(cvpb_context* ctx, const cvpb_cvp_options* opts,
                              const cvpb_exec_policy* exec, const double* proj, double* volume,
                              double* view_seconds);

/* view_seconds of the host calls (cvp.cpp:469-477 times each view's loop).
 * The device runs all views of a launch at once, so a launch's measured time
 * is attributed to its views in proportion to their work, the number of
 * voxel-column cuts each view has; this returns those weights for views
 * [view_begin, view_begin + view_count) (normalized to sum 1; equal weights
 * when no view has a cut). Builds the range's cut table when it is not
 * resident. Synchronous on the context's stream. */
int cvpb_cvp_view_weights(cvpb_context* ctx, const cvpb_cvp_options* opts, int view_begin,
                          int view_count, double* weights);

/* Multi-GPU building blocks of the host path (one rank per GPU, views
 * sharded: each rank's context holds its own view subset). The backward of
 * the host stack with the float32 partial volume left in d_volume (no D2H):
 * the caller sums partials across ranks (NCCL reduce-scatter over z-slabs)
 * and brings its slab back with cvpb_vec_to_host64. Asynchronous on `stream`. */
int cvpb_backproject_cvp_host_partial(cvpb_context* ctx, const cvpb_cvp_options* opts,
                                      const cvpb_exec_policy* exec, const double* proj,
                                      float* d_volume, void* stream);
/* float32 device vector -> float64 host buffer (pinned: written in place;
 * pageable: staged through the context). Synchronous. */
int cvpb_vec_to_host64(cvpb_context* ctx, const float* d_in, double* host, size_t n, void* stream);

/* collect_cut_records (cvp.cpp:652-689) evaluated by the DEVICE kernel's own
 * cut/row code for voxel (i,j,k) under view `view`; clamp = 0 reproduces the
 * reference (no detector clamping). Writes at most cap records, total in *n_out. */
int cvpb_collect_cut_records(cvpb_context* ctx, const cvpb_cvp_options* opts, int view, int i,
                             int j, int k, int clamp, int cap, int* rows, int* cols,
                             double* volume, double* inv_r2, int* n_out);
/* Device pixel-scale image of one view (float64 [rows][cols]) for checking. */
int cvpb_scale_image(cvpb_context* ctx, int view, int exact, double* out_host);

/* ---- Siddon-K (siddon.hpp:34-55) ---------------------------------------- */
int cvpb_project_siddon(cvpb_context* ctx, int k_per_edge, const cvpb_pixel_roi* roi,
                        const cvpb_exec_policy* exec, const float* d_volume, float* d_proj,
                        int view_begin, int view_count, void* stream);
int cvpb_backproject_siddon(cvpb_context* ctx, int k_per_edge, const cvpb_exec_policy* exec,
                            const float* d_proj, float* d_volume, int view_begin, int view_count,
                            int accumulate, void* stream);

/* trace_ray (siddon.cpp:154-164): the device traversal of one ray source ->
 * target through `vol`; writes at most cap (i, j, k) triples and chord
 * lengths [mm], total count in *n_out. */
int cvpb_trace_ray(cvpb_context* ctx, const cvpb_volume_geometry* vol, const double source[3],
                   const double target[3], int cap, int* ijk, double* length, int* n_out);

/* ---- TT footprint (new; see cvpb_tt_options) ----------------------------- */
int cvpb_project_tt(cvpb_context* ctx, const cvpb_tt_options* opts, const float* d_volume,
                    float* d_proj, int view_begin, int view_count, void* stream);
int cvpb_backproject_tt(cvpb_context* ctx, const cvpb_tt_options* opts, const float* d_proj,
                        float* d_volume, int view_begin, int view_count, int accumulate,
                        void* stream);

/* ---- reference-facing host paths for Siddon-K, TT and CGLS -------------------
 * float64 host buffers in the reference layout; conversion and copies happen
 * on the device inside the call (same contract as cvpb_project_cvp_host). */
int cvpb_project_siddon_host(cvpb_context* ctx, int k_per_edge, const cvpb_pixel_roi* roi,
                             const cvpb_exec_policy* exec, const double* volume, double* proj);
int cvpb_backproject_siddon_host(cvpb_context* ctx, int k_per_edge, const cvpb_exec_policy* exec,
                                 const double* proj, double* volume);
int cvpb_project_tt_host(cvpb_context* ctx, const cvpb_tt_options* opts, const double* volume,
                         double* proj);
int cvpb_backproject_tt_host(cvpb_context* ctx, const cvpb_tt_options* opts, const double* proj,
                             double* volume);
/* cgls (solver.cpp:55-106) device-resident, host data in / host iterate out. */
int cvpb_cgls_host(cvpb_context* ctx, int projector, const cvpb_cvp_options* cvp_opts,
                   const cvpb_tt_options* tt_opts, const cvpb_exec_policy* exec, int k_per_edge,
                   const double* b, double* x, int iterations, double* residual_norms);

/* ---- device vector ops for CGLS (solver.cpp:15-106) ---------------------- */
/* Compensated float64 dot of two float32 device vectors (dot_kahan,
 * solver.cpp:15-24); result written to *out_host after a stream sync. */
int cvpb_vec_dot(cvpb_context* ctx, const float* a, const float* b, size_t n, double* out_host,
                 void* stream);
/* y += alpha * x */
int cvpb_vec_axpy(cvpb_context* ctx, double alpha, const float* x, float* y, size_t n,
                  void* stream);
/* p = s + beta * p */
int cvpb_vec_xpby(cvpb_context* ctx, const float* s, double beta, float* p, size_t n,
                  void* stream);
/* 1 if every element is finite (cgls check_finite, solver.cpp:60-65). */
int cvpb_vec_all_finite(cvpb_context* ctx, const float* x, size_t n, int* out_host, void* stream);

/* SART / OS-SART pieces (PAPER.md:443-445 uses OS-SART with these
 * projectors): out = (b - ax) / rowsum where rowsum > eps,
 * else 0; x += lambda * corr / colsum where colsum > eps, clamped at 0 when
 * nonneg. */
int cvpb_vec_sart_residual(cvpb_context* ctx, const float* b, const float* ax, const float* rowsum,
                           float* out, size_t n, void* stream);
int cvpb_vec_sart_update(cvpb_context* ctx, float* x, const float* corr, const float* colsum,
                         double lambda, int nonneg, size_t n, void* stream);

/* Device-resident CGLS (cgls, solver.cpp:55-106) over the context's scene.
 * projector: 0 = CVP (cvp_opts), 1 = Siddon-K (k_per_edge), 2 = TT (tt_opts);
 * every operator call receives `exec` (NULL = ExecPolicy{}: Siddon K >= 128
 * is refused unless exec->allow_expensive, like the reference).
 * gamma / alpha / beta stay on the device (fused vector kernels); the host
 * reads a status word once per iteration for the reference's early exits.
 * d_b is the data (float32 stack, not modified), d_x receives the iterate;
 * residual_norms[iterations+1] receives ||b - A x_k|| (entry 0 = ||b||).
 * Scratch vectors are owned by the context. */
int cvpb_cgls(cvpb_context* ctx, int projector, const cvpb_cvp_options* cvp_opts,
              const cvpb_tt_options* tt_opts, const cvpb_exec_policy* exec, int k_per_edge,
              const float* d_b, float* d_x, int iterations, double* residual_norms, void* stream);

/* ---- multi-device scenes ------------------------------------
 * One process drives several GPUs: a group holds one context per member
 * device with the same scene. Views are sharded in contiguous ranges (member
 * g owns views [V g / N, V (g+1) / N)); the volume is sharded in contiguous
 * z-slabs (planes [N3 g / N, N3 (g+1) / N)), the k-slowest layout of
 * geometry.hpp:34-36 making each slab one contiguous range.
 *   forward   each member uploads its slab of the host volume, the slabs are
 *             all-gathered over NVLink (peer copies), and each member
 *             projects its views into its part of the host stack — no
 *             exchange of projections at all;
 *   backward  each member backprojects its views into a full partial volume,
 *             then reduce-scatters the partials over peer memory (one kernel
 *             per member reads its slab out of every member's partial, sums
 *             the members in a fixed order in float64) and writes its slab of
 *             the host volume.
 * Members may repeat a device (e.g. {0, 0}): the same code then runs with
 * every member on one GPU, which is how the multi-device path is tested on a
 * single-GPU box. With one member every call is the single-context call.
 * The reference entry points these replace for an unchanged C++ caller:
 * project_cvp_into / backproject_cvp_into (cvp.hpp:87-99) — the drop-in
 * (libcbct_b200) builds its scenes as groups over every visible GPU, or over
 * the devices listed in CBCT_B200_DEVICES (e.g. "0,0"). */
typedef struct cvpb_group cvpb_group;
/* devices == NULL or n_devices == 0: every visible device. At most 16 members. */
int cvpb_group_create(const int* devices, int n_devices, cvpb_group** out);
void cvpb_group_destroy(cvpb_group* g);
int cvpb_group_size(const cvpb_group* g, int* n_members);
/* member m's device, view shard and volume slab (elements) — after set_geometry */
int cvpb_group_member(const cvpb_group* g, int member, int* device, int* view_begin,
                      int* view_count, size_t* slab_begin, size_t* slab_count);
/* member m's context (single-device calls on the same scene, e.g. Siddon) */
int cvpb_group_context(cvpb_group* g, int member, cvpb_context** out);
int cvpb_group_set_geometry(cvpb_group* g, const cvpb_volume_geometry* vol,
                            const cvpb_detector_geometry* det, int n_views, const cvpb_view* views);
/* project_cvp_into / backproject_cvp_into over the group (float64 host
 * buffers, reference semantics; view_seconds[v] = the owning member's time
 * per view). */
int cvpb_group_project_cvp_host(cvpb_group* g, const cvpb_cvp_options* opts,
                                const cvpb_exec_policy* exec, const double* volume, double* proj,
                                double* view_seconds);
int cvpb_group_backproject_cvp_host(cvpb_group* g, const cvpb_cvp_options* opts,
                                    const cvpb_exec_policy* exec, const double* proj,
                                    double* volume, double* view_seconds);
int cvpb_group_project_tt_host(cvpb_group* g, const cvpb_tt_options* opts, const double* volume,
                               double* proj);
int cvpb_group_backproject_tt_host(cvpb_group* g, const cvpb_tt_options* opts, const double* proj,
                                   double* volume);
/* cgls (solver.cpp:55-106) device-resident across the group: per iteration
 * one sharded P (after an all-gather of the direction's slabs), one sharded
 * BP + peer reduce-scatter into slabs, slab-local vector updates; the dots
 * are summed over the members in a fixed order (float64). Same arguments and
 * early exits as cvpb_cgls_host. */
int cvpb_group_cgls_host(cvpb_group* g, int projector, const cvpb_cvp_options* cvp_opts,
                         const cvpb_tt_options* tt_opts, const cvpb_exec_policy* exec,
                         int k_per_edge, const double* b, double* x, int iterations,
                         double* residual_norms);

#ifdef __cplusplus
}
#endif
#endif /* CVPB200_H */
