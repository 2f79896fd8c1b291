// cbct_b200 — C++ drop-in for the reference's operator API.
//
// A caller of the reference library (cbctproj, /root/reference/proj/include/
// cbct/*.hpp) switches its include path to /root/repo/include (the one-line
// forwarders in include/cbct/ map every reference header here) and links
// libcbct_b200.so instead of libcbct.a. Types, function names, argument
// meaning, defaults and the exception type raised for each error condition are
// the reference's; the numeric work runs on the GPU through libcvpb200's C ABI
// (include/cvpb200.h). See INTEGRATION.md.
//
// Also provided (host float64, csrc/dropin/): the polygon kernel
// (cbct_b200/polygon.hpp), the CVP introspection helpers column_cuts,
// row_breakpoints and elevation_corrected_split (cvp.hpp:48-79), DEN I/O
// (cbct_b200/den.hpp) and logging (cbct_b200/log.hpp), so the reference's own
// callers — its unit tests and acceptance harness — compile unchanged.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <functional>
#include <random>
#include <span>
#include <stdexcept>
#include <vector>

#include "cbct_b200/polygon.hpp"
#include "cbct_b200/vec.hpp"

namespace cbct {

// ---- geometry (geometry.hpp) -------------------------------------------------
struct VolumeGeometry {
    std::array<int, 3> counts{};
    Vec3d voxel_size{};
    static VolumeGeometry make(std::array<int, 3> counts, Vec3d voxel_size);
    Vec3d extent() const {
        return {counts[0] * voxel_size.x, counts[1] * voxel_size.y, counts[2] * voxel_size.z};
    }
    Vec3d min_corner() const { return extent() * -0.5; }
    Vec3d voxel_center(int i, int j, int k) const;
    std::size_t voxel_count() const {
        return std::size_t(counts[0]) * std::size_t(counts[1]) * std::size_t(counts[2]);
    }
    std::size_t linear_index(int i, int j, int k) const {
        return (std::size_t(k) * counts[1] + std::size_t(j)) * counts[0] + std::size_t(i);
    }
    bool operator==(const VolumeGeometry&) const = default;
};

struct DetectorGeometry {
    int rows = 0;
    int cols = 0;
    double pixel_width = 1.0;
    double pixel_height = 1.0;
    static DetectorGeometry make(int rows, int cols, double pixel_width, double pixel_height);
    double pixel_area() const { return pixel_width * pixel_height; }
    Vec2d pixel_size() const { return {pixel_width, pixel_height}; }
    std::size_t pixel_count() const { return std::size_t(rows) * std::size_t(cols); }
    bool operator==(const DetectorGeometry&) const = default;
};

struct LocalSpherical {
    double r, theta, phi;
};

class ViewGeometry {
  public:
    static ViewGeometry make(const Vec3d& source, const Mat3d& frame, double focal_length,
                             const Vec2d& principal_point, const Vec2d& pixel_size);
    const Vec3d& source() const { return source_; }
    const Mat3d& frame() const { return frame_; }
    double focal_length() const { return f_; }
    const Vec2d& principal_point() const { return pp_; }
    const Vec2d& pixel_size() const { return b_; }
    const Mat3d& camera_matrix() const { return cam_; }
    Vec2d project_point(const Vec3d& x) const;
    double depth(const Vec3d& x) const { return dot(frame_.row(2), x - source_); }
    LocalSpherical to_local_spherical(const Vec3d& x) const;
    double elevation_angle(const Vec2d& chi) const;
    Vec3d detector_point(const Vec2d& chi) const;
    std::array<double, 12> standard_matrix() const;
    static ViewGeometry from_standard_matrix(const std::array<double, 12>& P, const Vec2d& pixel_size);

  private:
    ViewGeometry() = default;
    Vec3d source_{};
    Mat3d frame_{};
    double f_ = 0.0;
    Vec2d pp_{}, b_{};
    Mat3d cam_{};
};

std::vector<ViewGeometry> make_circular_trajectory(double sid, double sdd, int n_views,
                                                   double arc_deg, const DetectorGeometry& det);
void write_camera_matrices(const std::filesystem::path& path, std::span<const ViewGeometry> views);
std::vector<ViewGeometry> read_camera_matrices(const std::filesystem::path& path,
                                               const Vec2d& pixel_size);

// ---- data containers (volume.hpp) -------------------------------------------------
struct AttenuationVolume {
    VolumeGeometry geom;
    std::vector<double> values;
    static AttenuationVolume zeros(const VolumeGeometry& g) {
        return {g, std::vector<double>(g.voxel_count(), 0.0)};
    }
    double& at(int i, int j, int k) { return values[geom.linear_index(i, j, k)]; }
    double at(int i, int j, int k) const { return values[geom.linear_index(i, j, k)]; }
};

struct ProjectionStack {
    DetectorGeometry det;
    int n_views = 0;
    std::vector<double> values;
    static ProjectionStack zeros(const DetectorGeometry& d, int n_views) {
        return {d, n_views, std::vector<double>(d.pixel_count() * std::size_t(n_views), 0.0)};
    }
    std::size_t view_size() const { return det.pixel_count(); }
    std::span<double> view(int v) { return {values.data() + view_size() * v, view_size()}; }
    std::span<const double> view(int v) const { return {values.data() + view_size() * v, view_size()}; }
    double& at(int v, int m, int n) { return values[view_size() * v + std::size_t(m) * det.cols + n]; }
    double at(int v, int m, int n) const { return values[view_size() * v + std::size_t(m) * det.cols + n]; }
};

// ---- execution policy (exec.hpp) ------------------------------------------------------
struct ExecPolicy {
    int threads = 0;             // ignored on the device
    bool deterministic = false;  // bit-reproducible backprojection (see cvpb200.h)
    bool allow_expensive = false;
    bool serial() const { return deterministic || threads == 1; }
};

// ---- CVP (cvp.hpp) ----------------------------------------------------------------------
enum class PixelScaling { Cos, Exact };
enum class CvpPrecision { Double, Single };
enum class RadiusEstimate { VoxelCenter, CutCentroid };

struct CvpOptions {
    PixelScaling scaling = PixelScaling::Exact;
    bool elevation_correction = true;
    CvpPrecision precision = CvpPrecision::Double;
    RadiusEstimate r_estimate = RadiusEstimate::CutCentroid;
};

struct CutVolumeRecord {
    int row = 0;
    int column = 0;
    double volume = 0.0;
    double inv_r2 = 0.0;
};

// Introspection (cvp.hpp:24-79): the cut of a voxel base by one detector
// column's boundary pre-images, and the z split of a vertical segment over
// detector rows (plain and elevation-corrected).
struct ColumnCut {
    int column = 0;
    Polygon2D polygon;
    double area = 0.0;
    Vec2d centroid{};
};

struct RowSegment {
    int row = 0;
    double length = 0.0;
};

std::vector<ColumnCut> column_cuts(const ViewGeometry& view, const DetectorGeometry& det,
                                   const Polygon2D& voxel_base);
std::vector<RowSegment> row_breakpoints(const ViewGeometry& view, const DetectorGeometry& det,
                                        const Vec2d& centroid, double z_lo, double z_hi);
inline double cut_volume(const ColumnCut& cut, double d) { return cut.area * d; }
std::vector<RowSegment> elevation_corrected_split(const ViewGeometry& view,
                                                  const DetectorGeometry& det,
                                                  const ColumnCut& cut, double z_lo, double z_hi,
                                                  double elevation);

double pixel_scale_cos(const ViewGeometry& view, const DetectorGeometry& det, int m, int n);
double spherical_quad_area(const Vec3d& t0, const Vec3d& t1, const Vec3d& t2, const Vec3d& t3);
double pixel_scale_exact(const ViewGeometry& view, const DetectorGeometry& det, int m, int n);

ProjectionStack project_cvp(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                            const DetectorGeometry& det, const CvpOptions& opts = {},
                            const ExecPolicy& exec = {});
void project_cvp_into(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                      const DetectorGeometry& det, const CvpOptions& opts, const ExecPolicy& exec,
                      ProjectionStack& out, std::vector<double>* view_seconds = nullptr);
AttenuationVolume backproject_cvp(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                                  const VolumeGeometry& vol_geom, const CvpOptions& opts = {},
                                  const ExecPolicy& exec = {});
void backproject_cvp_into(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                          const VolumeGeometry& vol_geom, const CvpOptions& opts,
                          const ExecPolicy& exec, AttenuationVolume& out,
                          std::vector<double>* view_seconds = nullptr);
std::vector<CutVolumeRecord> collect_cut_records(const VolumeGeometry& vol_geom,
                                                 const ViewGeometry& view,
                                                 const DetectorGeometry& det,
                                                 const CvpOptions& opts, int i, int j, int k);

// ---- Siddon-K (siddon.hpp) ----------------------------------------------------------------
struct RayIntersection {
    int i, j, k;
    double length;
};
using RayIntersectionList = std::vector<RayIntersection>;
RayIntersectionList trace_ray(const VolumeGeometry& vol, const Vec3d& source, const Vec3d& target);

struct PixelRoi {
    int row_begin = 0;
    int row_end = -1;
    int col_begin = 0;
    int col_end = -1;
};

ProjectionStack project_siddon_k(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                                 const DetectorGeometry& det, int k_per_edge,
                                 const ExecPolicy& exec = {});
void project_siddon_k_into(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                           const DetectorGeometry& det, int k_per_edge, const ExecPolicy& exec,
                           ProjectionStack& out, const PixelRoi& roi = {},
                           std::vector<double>* view_seconds = nullptr);
AttenuationVolume backproject_siddon_k(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                                       const VolumeGeometry& vol_geom, int k_per_edge,
                                       const ExecPolicy& exec = {});
void backproject_siddon_k_into(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                               const VolumeGeometry& vol_geom, int k_per_edge,
                               const ExecPolicy& exec, AttenuationVolume& out,
                               std::vector<double>* view_seconds = nullptr);

// ---- solver (solver.hpp) ----------------------------------------------------------------------
struct LinearOperatorPair {
    std::function<void(const AttenuationVolume&, ProjectionStack&)> forward;
    std::function<void(const ProjectionStack&, AttenuationVolume&)> adjoint;
    VolumeGeometry vol_geom;
    DetectorGeometry det;
    int n_views = 0;
    std::size_t domain_size() const { return vol_geom.voxel_count(); }
    std::size_t range_size() const { return det.pixel_count() * std::size_t(n_views); }
};

inline double uniform01(std::mt19937_64& rng) { return double(rng() >> 11) * 0x1.0p-53; }
void fill_uniform01(std::span<double> out, std::uint64_t seed);
double adjoint_test(const LinearOperatorPair& pair, std::uint64_t seed);

struct CglsResult {
    AttenuationVolume x;
    std::vector<double> residual_norms;
};
CglsResult cgls(const LinearOperatorPair& pair, ProjectionStack b, int iterations);
double relative_projector_error(std::span<const double> view, std::span<const double> view_ref);
double extinction_from_intensity(double I0, double I);

// ---- B200 extensions ---------------------------------------------------------------------------
namespace b200 {

// TT separable-footprint pair (no reference symbol; see cvpb200.h).
enum class TTAmplitude { A1 = 0, A2 = 1 };
ProjectionStack project_tt(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                           const DetectorGeometry& det, TTAmplitude amp = TTAmplitude::A2);
AttenuationVolume backproject_tt(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                                 const VolumeGeometry& vol_geom, TTAmplitude amp = TTAmplitude::A2);

// Operator pairs whose forward/adjoint run on the GPU; pairs built here also
// let cgls_device run the whole recurrence device-resident (cvpb_cgls).
LinearOperatorPair cvp_pair(const VolumeGeometry& vol, const DetectorGeometry& det,
                            std::span<const ViewGeometry> views, const CvpOptions& opts = {});
LinearOperatorPair siddon_pair(const VolumeGeometry& vol, const DetectorGeometry& det,
                               std::span<const ViewGeometry> views, int k_per_edge);
CglsResult cgls_device(const VolumeGeometry& vol, const DetectorGeometry& det,
                       std::span<const ViewGeometry> views, const CvpOptions& opts,
                       const ProjectionStack& b, int iterations);

}  // namespace b200

}  // namespace cbct
