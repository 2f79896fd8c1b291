// libcbct_b200.so — the reference's C++ operator API (namespace cbct) over the
// libcvpb200 C ABI. Every operator call goes to the GPU; this file only maps
// types, validates shapes like the reference, caches device scenes, and turns
// C-ABI status codes back into the reference's exception types.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <list>
#include <memory>
#include <mutex>
#include <numbers>
#include <sstream>
#include <string>

#include "cbct_b200/cbct.hpp"
#include "cvpb200.h"

namespace cbct {

namespace {

[[noreturn]] void throw_status(int rc) {
    const std::string msg = cvpb_last_error();
    switch (rc) {
        case CVPB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case CVPB_OUT_OF_RANGE: throw std::out_of_range(msg);
        case CVPB_DOMAIN_ERROR: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

void check(int rc) {
    if (rc != CVPB_OK) throw_status(rc);
}

cvpb_view to_c(const ViewGeometry& v) {
    cvpb_view c;
    c.source[0] = v.source().x;
    c.source[1] = v.source().y;
    c.source[2] = v.source().z;
    std::memcpy(c.frame, v.frame().m.data(), sizeof c.frame);
    c.focal_length = v.focal_length();
    c.principal_point[0] = v.principal_point().x;
    c.principal_point[1] = v.principal_point().y;
    c.pixel_size[0] = v.pixel_size().x;
    c.pixel_size[1] = v.pixel_size().y;
    return c;
}

cvpb_volume_geometry to_c(const VolumeGeometry& g) {
    return {{g.counts[0], g.counts[1], g.counts[2]}, {g.voxel_size.x, g.voxel_size.y, g.voxel_size.z}};
}

cvpb_detector_geometry to_c(const DetectorGeometry& d) {
    return {d.rows, d.cols, d.pixel_width, d.pixel_height};
}

cvpb_cvp_options to_c(const CvpOptions& o) {
    return {o.scaling == PixelScaling::Exact ? 1 : 0, o.elevation_correction ? 1 : 0,
            o.precision == CvpPrecision::Single ? 1 : 0,
            o.r_estimate == RadiusEstimate::CutCentroid ? 1 : 0};
}

cvpb_exec_policy to_c(const ExecPolicy& e) {
    return {e.threads, e.deterministic ? 1 : 0, e.allow_expensive ? 1 : 0};
}

// Device scenes keyed by (volume, detector, views); a small LRU so repeated
// calls with the same geometry (CGLS, benchmarks) reuse the resident views and
// pixel-scale images. The reference's free functions are reentrant, so each
// call holds a Lease: a shared_ptr that keeps its entry alive even if the LRU
// evicts it meanwhile, plus the entry's mutex for the whole call (a context's
// host-path buffers, cut-table key and scratch are mutable state). Calls on
// different scenes run concurrently; calls on one scene serialise.
//
// A scene is a multi-device group (cvpb_group, include/cvpb200.h) over every
// visible GPU — or the devices listed in CBCT_B200_DEVICES ("0,1,2,3", or
// "0,0" for two members on one GPU) — so an unchanged caller of
// project_cvp_into / backproject_cvp_into / cgls runs view-sharded on all of
// them; with one device the group is the single-context path. Siddon-K and
// the introspection calls run on member 0's context.
struct SceneEntry {
    cvpb_volume_geometry vol;
    cvpb_detector_geometry det;
    std::vector<cvpb_view> views;
    cvpb_group* grp = nullptr;
    cvpb_context* ctx = nullptr;  // member 0 (owned by the group)
    std::mutex mu;
    ~SceneEntry() {
        if (grp) cvpb_group_destroy(grp);
    }
};

struct Lease {
    std::shared_ptr<SceneEntry> entry;
    std::unique_lock<std::mutex> lock;
    cvpb_context* get() const { return entry->ctx; }
    operator cvpb_context*() const { return entry->ctx; }
    cvpb_group* group() const { return entry->grp; }
};

// CBCT_B200_DEVICES="i,j,..." -> member devices; empty = every visible device
std::vector<int> group_devices() {
    std::vector<int> out;
    if (const char* env = std::getenv("CBCT_B200_DEVICES")) {
        std::stringstream ss(env);
        std::string tok;
        while (std::getline(ss, tok, ','))
            if (!tok.empty()) out.push_back(std::stoi(tok));
    }
    return out;
}

std::mutex g_mu;  // guards the LRU list only
std::list<std::shared_ptr<SceneEntry>> g_scenes;

bool same(const SceneEntry& e, const cvpb_volume_geometry& v, const cvpb_detector_geometry& d,
          const std::vector<cvpb_view>& views) {
    return std::memcmp(&e.vol, &v, sizeof v) == 0 && std::memcmp(&e.det, &d, sizeof d) == 0 &&
           e.views.size() == views.size() &&
           (views.empty() || std::memcmp(e.views.data(), views.data(), sizeof(cvpb_view) * views.size()) == 0);
}

Lease scene(const VolumeGeometry& vg, const DetectorGeometry& dg, std::span<const ViewGeometry> views) {
    const cvpb_volume_geometry v = to_c(vg);
    const cvpb_detector_geometry d = to_c(dg);
    std::vector<cvpb_view> cv;
    cv.reserve(views.size());
    for (const auto& x : views) cv.push_back(to_c(x));
    std::shared_ptr<SceneEntry> e;
    {
        std::lock_guard<std::mutex> lock(g_mu);
        for (auto it = g_scenes.begin(); it != g_scenes.end(); ++it)
            if (same(**it, v, d, cv)) {
                g_scenes.splice(g_scenes.begin(), g_scenes, it);
                e = g_scenes.front();
                break;
            }
    }
    if (!e) {
        // build outside the list lock (uploads views, scale images); a racing
        // thread may build the same scene, the list then holds both for a while
        e = std::make_shared<SceneEntry>();
        e->vol = v;
        e->det = d;
        e->views = cv;
        const std::vector<int> devs = group_devices();
        check(cvpb_group_create(devs.empty() ? nullptr : devs.data(), int(devs.size()), &e->grp));
        check(cvpb_group_set_geometry(e->grp, &v, &d, int(cv.size()), cv.data()));
        check(cvpb_group_context(e->grp, 0, &e->ctx));
        std::lock_guard<std::mutex> lock(g_mu);
        g_scenes.push_front(e);
        while (g_scenes.size() > 4) g_scenes.pop_back();  // leases keep evicted entries alive
    }
    Lease l{e, std::unique_lock<std::mutex>(e->mu)};
    return l;
}

// geometry-less context for trace_ray (its scratch is per context: one caller at a time)
Lease any_context() {
    static std::shared_ptr<SceneEntry> e = [] {
        auto p = std::make_shared<SceneEntry>();
        const int dev0 = 0;
        check(cvpb_group_create(&dev0, 1, &p->grp));
        check(cvpb_group_context(p->grp, 0, &p->ctx));
        return p;
    }();
    return Lease{e, std::unique_lock<std::mutex>(e->mu)};
}

ViewGeometry from_c(const cvpb_view& c);

double dot_kahan(std::span<const double> a, std::span<const double> b) {
    double sum = 0.0, comp = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double y = a[i] * b[i] - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    return sum;
}

}  // namespace

// ---- geometry -------------------------------------------------------------------

// VolumeGeometry::make / voxel_center and DetectorGeometry::make restate
// geometry.cpp:23-48 (same checks and messages: the exception contract).
VolumeGeometry VolumeGeometry::make(std::array<int, 3> counts, Vec3d voxel_size) {
    for (int c : counts)
        if (c <= 0) throw std::invalid_argument("voxel counts must be positive");
    for (double a : {voxel_size.x, voxel_size.y, voxel_size.z}) {
        if (!std::isfinite(a)) throw std::invalid_argument("voxel size is not finite");
        if (a <= 0.0) throw std::invalid_argument("voxel sizes must be positive");
    }
    return {counts, voxel_size};
}

Vec3d VolumeGeometry::voxel_center(int i, int j, int k) const {
    if (i < 0 || j < 0 || k < 0 || i >= counts[0] || j >= counts[1] || k >= counts[2])
        throw std::out_of_range("voxel index outside lattice");
    const Vec3d l = extent();
    return {(voxel_size.x - l.x) * 0.5 + i * voxel_size.x, (voxel_size.y - l.y) * 0.5 + j * voxel_size.y,
            (voxel_size.z - l.z) * 0.5 + k * voxel_size.z};
}

DetectorGeometry DetectorGeometry::make(int rows, int cols, double pixel_width, double pixel_height) {
    if (rows <= 0 || cols <= 0) throw std::invalid_argument("detector counts must be positive");
    for (double b : {pixel_width, pixel_height}) {
        if (!std::isfinite(b)) throw std::invalid_argument("pixel size is not finite");
        if (b <= 0.0) throw std::invalid_argument("pixel sizes must be positive");
    }
    return {rows, cols, pixel_width, pixel_height};
}

namespace {
ViewGeometry from_c(const cvpb_view& c) {
    Mat3d fr;
    std::memcpy(fr.m.data(), c.frame, sizeof c.frame);
    return ViewGeometry::make({c.source[0], c.source[1], c.source[2]}, fr, c.focal_length,
                              {c.principal_point[0], c.principal_point[1]},
                              {c.pixel_size[0], c.pixel_size[1]});
}
}  // namespace

ViewGeometry ViewGeometry::make(const Vec3d& source, const Mat3d& frame, double focal_length,
                                const Vec2d& principal_point, const Vec2d& pixel_size) {
    const double s[3] = {source.x, source.y, source.z};
    const double pp[2] = {principal_point.x, principal_point.y};
    const double b[2] = {pixel_size.x, pixel_size.y};
    cvpb_view c;
    check(cvpb_view_make(s, frame.m.data(), focal_length, pp, b, &c));
    ViewGeometry g;
    g.source_ = {c.source[0], c.source[1], c.source[2]};
    std::memcpy(g.frame_.m.data(), c.frame, sizeof c.frame);
    g.f_ = c.focal_length;
    g.pp_ = {c.principal_point[0], c.principal_point[1]};
    g.b_ = {c.pixel_size[0], c.pixel_size[1]};
    double P[12];
    check(cvpb_view_standard_matrix(&c, P));
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) g.cam_(r, k) = P[4 * r + k];
    return g;
}

Vec2d ViewGeometry::project_point(const Vec3d& x) const {
    const cvpb_view c = to_c(*this);
    const double p[3] = {x.x, x.y, x.z};
    double chi[2];
    check(cvpb_view_project_point(&c, p, chi));
    return {chi[0], chi[1]};
}

// to_local_spherical / elevation_angle / detector_point: geometry.cpp:98-118.
LocalSpherical ViewGeometry::to_local_spherical(const Vec3d& x) const {
    const Vec3d d = x - source_;
    const double r = norm(d);
    if (!(r > 0.0)) throw std::domain_error("point coincides with the source");
    const Vec3d local = frame_ * d;
    const double theta = std::acos(std::clamp(local.z / r, -1.0, 1.0));
    double phi = std::atan2(local.y, local.x);
    if (phi < 0.0) phi += 2.0 * std::numbers::pi;
    return {r, theta, phi};
}

double ViewGeometry::elevation_angle(const Vec2d& chi) const {
    const double u = (chi.x - pp_.x) * b_.x, v = (chi.y - pp_.y) * b_.y;
    return std::atan2(std::abs(v), std::hypot(u, f_));
}

Vec3d ViewGeometry::detector_point(const Vec2d& chi) const {
    const Vec3d local{(chi.x - pp_.x) * b_.x, (chi.y - pp_.y) * b_.y, f_};
    return source_ + frame_.transposed() * local;
}

std::array<double, 12> ViewGeometry::standard_matrix() const {
    const cvpb_view c = to_c(*this);
    std::array<double, 12> P;
    check(cvpb_view_standard_matrix(&c, P.data()));
    return P;
}

ViewGeometry ViewGeometry::from_standard_matrix(const std::array<double, 12>& P,
                                                const Vec2d& pixel_size) {
    const double b[2] = {pixel_size.x, pixel_size.y};
    cvpb_view c;
    check(cvpb_view_from_standard_matrix(P.data(), b, &c));
    return from_c(c);
}

std::vector<ViewGeometry> make_circular_trajectory(double sid, double sdd, int n_views,
                                                   double arc_deg, const DetectorGeometry& det) {
    if (n_views <= 0) throw std::invalid_argument("need at least one view");
    std::vector<cvpb_view> c(n_views);
    const cvpb_detector_geometry d = to_c(det);
    check(cvpb_make_circular_trajectory(sid, sdd, n_views, arc_deg, &d, c.data()));
    std::vector<ViewGeometry> out;
    out.reserve(n_views);
    for (const auto& v : c) out.push_back(from_c(v));
    return out;
}

// Camera-matrix text I/O: geometry.cpp:212-249 (17 significant digits, '#'
// comments, the reference's error texts).
void write_camera_matrices(const std::filesystem::path& path, std::span<const ViewGeometry> views) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open " + path.string() + " for writing");
    out.precision(17);
    for (const ViewGeometry& v : views) {
        const auto P = v.standard_matrix();
        for (int i = 0; i < 12; ++i) out << P[i] << (i == 11 ? '\n' : ' ');
    }
    if (!out) throw std::runtime_error("failed writing " + path.string());
}

std::vector<ViewGeometry> read_camera_matrices(const std::filesystem::path& path,
                                               const Vec2d& pixel_size) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path.string());
    std::vector<ViewGeometry> views;
    std::string line;
    std::size_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        const auto first = line.find_first_not_of(" \t\r");
        if (first == std::string::npos || line[first] == '#') continue;
        std::istringstream ls(line);
        std::array<double, 12> P;
        for (double& e : P)
            if (!(ls >> e))
                throw std::runtime_error(path.string() + ":" + std::to_string(lineno) +
                                         ": expected 12 numbers per line");
        double extra;
        if (ls >> extra)
            throw std::runtime_error(path.string() + ":" + std::to_string(lineno) +
                                     ": expected 12 numbers per line");
        views.push_back(ViewGeometry::from_standard_matrix(P, pixel_size));
    }
    if (views.empty()) throw std::runtime_error(path.string() + ": no matrices found");
    return views;
}

// ---- CVP -----------------------------------------------------------------------------

double pixel_scale_cos(const ViewGeometry& view, const DetectorGeometry& det, int m, int n) {
    const cvpb_view c = to_c(view);
    const cvpb_detector_geometry d = to_c(det);
    double out;
    check(cvpb_pixel_scale(&c, &d, 0, m, n, &out));
    return out;
}

double pixel_scale_exact(const ViewGeometry& view, const DetectorGeometry& det, int m, int n) {
    const cvpb_view c = to_c(view);
    const cvpb_detector_geometry d = to_c(det);
    double out;
    check(cvpb_pixel_scale(&c, &d, 1, m, n, &out));
    return out;
}

// spherical_quad_area: cvp.cpp:580-599 (edge-normal form and domain checks of
// the public helper; the device scale images use a cancellation-free form).
double spherical_quad_area(const Vec3d& t0, const Vec3d& t1, const Vec3d& t2, const Vec3d& t3) {
    const Vec3d t[4] = {t0, t1, t2, t3};
    for (const Vec3d& v : t)
        if (std::abs(norm(v) - 1.0) > 1e-12)
            throw std::invalid_argument("spherical quad vertices must be unit vectors");
    Vec3d nrm[4];
    for (int i = 0; i < 4; ++i) {
        nrm[i] = cross(t[i], t[(i + 1) % 4]);
        if (squared_norm(nrm[i]) < 1e-30)
            throw std::domain_error("degenerate spherical quad (parallel consecutive vertices)");
        nrm[i] = nrm[i] / norm(nrm[i]);
    }
    double sum = 0.0;
    for (int i = 0; i < 4; ++i) sum += std::acos(std::clamp(dot(nrm[i], nrm[(i + 1) % 4]), -1.0, 1.0));
    const double area = 2.0 * std::numbers::pi - sum;
    if (!(area > 0.0) || !(area < 4.0 * std::numbers::pi))
        throw std::domain_error("spherical quad area outside (0, 4*pi)");
    return area;
}

void project_cvp_into(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                      const DetectorGeometry& det, const CvpOptions& opts, const ExecPolicy& exec,
                      ProjectionStack& out, std::vector<double>* view_seconds) {
    if (out.det != det || out.n_views != int(views.size()))
        throw std::invalid_argument("output stack does not match detector/views");
    if (view_seconds) view_seconds->assign(views.size(), 0.0);
    Lease ctx = scene(vol.geom, det, views);
    const cvpb_cvp_options o = to_c(opts);
    const cvpb_exec_policy e = to_c(exec);
    check(cvpb_group_project_cvp_host(ctx.group(), &o, &e, vol.values.data(), out.values.data(),
                                      view_seconds ? view_seconds->data() : nullptr));
}

ProjectionStack project_cvp(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                            const DetectorGeometry& det, const CvpOptions& opts,
                            const ExecPolicy& exec) {
    ProjectionStack out = ProjectionStack::zeros(det, int(views.size()));
    project_cvp_into(vol, views, det, opts, exec, out);
    return out;
}

void backproject_cvp_into(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                          const VolumeGeometry& vol_geom, const CvpOptions& opts,
                          const ExecPolicy& exec, AttenuationVolume& out,
                          std::vector<double>* view_seconds) {
    if (out.geom != vol_geom) throw std::invalid_argument("output volume does not match geometry");
    if (proj.n_views != int(views.size()))
        throw std::invalid_argument("projection stack does not match views");
    if (view_seconds) view_seconds->assign(views.size(), 0.0);
    Lease ctx = scene(vol_geom, proj.det, views);
    const cvpb_cvp_options o = to_c(opts);
    const cvpb_exec_policy e = to_c(exec);
    check(cvpb_group_backproject_cvp_host(ctx.group(), &o, &e, proj.values.data(), out.values.data(),
                                          view_seconds ? view_seconds->data() : nullptr));
}

AttenuationVolume backproject_cvp(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                                  const VolumeGeometry& vol_geom, const CvpOptions& opts,
                                  const ExecPolicy& exec) {
    AttenuationVolume out = AttenuationVolume::zeros(vol_geom);
    backproject_cvp_into(proj, views, vol_geom, opts, exec, out);
    return out;
}

std::vector<CutVolumeRecord> collect_cut_records(const VolumeGeometry& vol_geom,
                                                 const ViewGeometry& view,
                                                 const DetectorGeometry& det,
                                                 const CvpOptions& opts, int i, int j, int k) {
    if (i < 0 || j < 0 || k < 0 || i >= vol_geom.counts[0] || j >= vol_geom.counts[1] ||
        k >= vol_geom.counts[2])
        throw std::out_of_range("voxel index outside lattice");
    Lease ctx = scene(vol_geom, det, std::span<const ViewGeometry>(&view, 1));
    const cvpb_cvp_options o = to_c(opts);
    int cap = 64, n = 0;
    for (;;) {
        std::vector<int> rows(cap), cols(cap);
        std::vector<double> vol(cap), inv(cap);
        check(cvpb_collect_cut_records(ctx, &o, 0, i, j, k, 0, cap, rows.data(), cols.data(),
                                       vol.data(), inv.data(), &n));
        if (n <= cap) {
            std::vector<CutVolumeRecord> out(n);
            for (int t = 0; t < n; ++t) out[t] = {rows[t], cols[t], vol[t], inv[t]};
            return out;
        }
        cap = n;
    }
}

// ---- Siddon-K ------------------------------------------------------------------------------

RayIntersectionList trace_ray(const VolumeGeometry& vol, const Vec3d& source, const Vec3d& target) {
    const cvpb_volume_geometry v = to_c(vol);
    const double s[3] = {source.x, source.y, source.z}, t[3] = {target.x, target.y, target.z};
    int cap = 4 * (vol.counts[0] + vol.counts[1] + vol.counts[2]) + 8, n = 0;
    std::vector<int> ijk(3 * cap);
    std::vector<double> len(cap);
    Lease ctx = any_context();
    check(cvpb_trace_ray(ctx, &v, s, t, cap, ijk.data(), len.data(), &n));
    RayIntersectionList out(std::min(n, cap));
    for (std::size_t q = 0; q < out.size(); ++q)
        out[q] = {ijk[3 * q], ijk[3 * q + 1], ijk[3 * q + 2], len[q]};
    return out;
}

void project_siddon_k_into(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                           const DetectorGeometry& det, int k_per_edge, const ExecPolicy& exec,
                           ProjectionStack& out, const PixelRoi& roi,
                           std::vector<double>* view_seconds) {
    if (out.det != det || out.n_views != int(views.size()))
        throw std::invalid_argument("output stack does not match detector/views");
    if (view_seconds) view_seconds->assign(views.size(), 0.0);
    Lease ctx = scene(vol.geom, det, views);
    const cvpb_exec_policy e = to_c(exec);
    const cvpb_pixel_roi r{roi.row_begin, roi.row_end, roi.col_begin, roi.col_end};
    check(cvpb_project_siddon_host(ctx, k_per_edge, &r, &e, vol.values.data(), out.values.data()));
}

ProjectionStack project_siddon_k(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                                 const DetectorGeometry& det, int k_per_edge, const ExecPolicy& exec) {
    ProjectionStack out = ProjectionStack::zeros(det, int(views.size()));
    project_siddon_k_into(vol, views, det, k_per_edge, exec, out);
    return out;
}

void backproject_siddon_k_into(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                               const VolumeGeometry& vol_geom, int k_per_edge,
                               const ExecPolicy& exec, AttenuationVolume& out,
                               std::vector<double>* view_seconds) {
    if (out.geom != vol_geom) throw std::invalid_argument("output volume does not match geometry");
    if (proj.n_views != int(views.size()))
        throw std::invalid_argument("projection stack does not match views");
    if (view_seconds) view_seconds->assign(views.size(), 0.0);
    Lease ctx = scene(vol_geom, proj.det, views);
    const cvpb_exec_policy e = to_c(exec);
    check(cvpb_backproject_siddon_host(ctx, k_per_edge, &e, proj.values.data(), out.values.data()));
}

AttenuationVolume backproject_siddon_k(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                                       const VolumeGeometry& vol_geom, int k_per_edge,
                                       const ExecPolicy& exec) {
    AttenuationVolume out = AttenuationVolume::zeros(vol_geom);
    backproject_siddon_k_into(proj, views, vol_geom, k_per_edge, exec, out);
    return out;
}

// ---- solver ------------------------------------------------------------------------------------

void fill_uniform01(std::span<double> out, std::uint64_t seed) {
    check(cvpb_fill_uniform01(out.data(), out.size(), seed));
}

// Generic solvers over the caller's std::function operators, with the
// reference's recurrences and compensated dots (solver.cpp:35-106). Pairs
// from b200::cvp_pair run their operators on the GPU; b200::cgls_device runs
// the recurrence itself device-resident.
double adjoint_test(const LinearOperatorPair& pair, std::uint64_t seed) {
    AttenuationVolume x = AttenuationVolume::zeros(pair.vol_geom);
    ProjectionStack b = ProjectionStack::zeros(pair.det, pair.n_views);
    std::mt19937_64 rng(seed);
    for (double& v : x.values) v = uniform01(rng);
    for (double& v : b.values) v = uniform01(rng);
    ProjectionStack ax = ProjectionStack::zeros(pair.det, pair.n_views);
    pair.forward(x, ax);
    AttenuationVolume atb = AttenuationVolume::zeros(pair.vol_geom);
    pair.adjoint(b, atb);
    const double lhs = dot_kahan(b.values, ax.values), rhs = dot_kahan(x.values, atb.values);
    const double den = std::max(std::abs(lhs), std::abs(rhs));
    if (den == 0.0) return std::numeric_limits<double>::quiet_NaN();
    return std::abs(lhs - rhs) / den;
}

CglsResult cgls(const LinearOperatorPair& pair, ProjectionStack b, int iterations) {
    if (iterations < 1) throw std::invalid_argument("cgls needs at least one iteration");
    if (b.det != pair.det || b.n_views != pair.n_views)
        throw std::invalid_argument("cgls data does not match the operator range");
    auto finite = [](std::span<const double> v, int it) {
        for (double x : v)
            if (!std::isfinite(x))
                throw std::runtime_error("CGLS diverged (non-finite iterate) at iteration " +
                                         std::to_string(it));
    };
    CglsResult res;
    res.x = AttenuationVolume::zeros(pair.vol_geom);
    ProjectionStack& r = b;
    res.residual_norms.push_back(std::sqrt(dot_kahan(r.values, r.values)));
    AttenuationVolume s = AttenuationVolume::zeros(pair.vol_geom);
    pair.adjoint(r, s);
    AttenuationVolume p = s;
    ProjectionStack q = ProjectionStack::zeros(pair.det, pair.n_views);
    double gamma = dot_kahan(s.values, s.values);
    for (int it = 1; it <= iterations; ++it) {
        if (gamma == 0.0) {
            res.residual_norms.push_back(res.residual_norms.back());
            continue;
        }
        pair.forward(p, q);
        const double qq = dot_kahan(q.values, q.values);
        if (qq == 0.0)
            throw std::runtime_error("CGLS breakdown (A p = 0) at iteration " + std::to_string(it));
        const double alpha = gamma / qq;
        for (std::size_t i = 0; i < res.x.values.size(); ++i) res.x.values[i] += alpha * p.values[i];
        for (std::size_t i = 0; i < r.values.size(); ++i) r.values[i] -= alpha * q.values[i];
        pair.adjoint(r, s);
        const double gamma_new = dot_kahan(s.values, s.values);
        const double beta = gamma_new / gamma;
        for (std::size_t i = 0; i < p.values.size(); ++i) p.values[i] = s.values[i] + beta * p.values[i];
        gamma = gamma_new;
        finite(res.x.values, it);
        finite(r.values, it);
        res.residual_norms.push_back(std::sqrt(dot_kahan(r.values, r.values)));
    }
    return res;
}

double relative_projector_error(std::span<const double> view, std::span<const double> view_ref) {
    if (view.size() != view_ref.size()) throw std::invalid_argument("view dimensions do not match");
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < view.size(); ++i) {
        const double d = view[i] - view_ref[i];
        num += d * d;
        den += view_ref[i] * view_ref[i];
    }
    if (den == 0.0) throw std::domain_error("reference view has zero norm");
    return 100.0 * std::sqrt(num / den);
}

double extinction_from_intensity(double I0, double I) {
    if (!(I0 > 0.0) || !(I > 0.0)) throw std::domain_error("intensities must be positive");
    return std::log(I0) - std::log(I);
}

// ---- B200 extensions ------------------------------------------------------------------------------

namespace b200 {

ProjectionStack project_tt(const AttenuationVolume& vol, std::span<const ViewGeometry> views,
                           const DetectorGeometry& det, TTAmplitude amp) {
    ProjectionStack out = ProjectionStack::zeros(det, int(views.size()));
    Lease ctx = scene(vol.geom, det, views);
    const cvpb_tt_options o{int(amp)};
    check(cvpb_group_project_tt_host(ctx.group(), &o, vol.values.data(), out.values.data()));
    return out;
}

AttenuationVolume backproject_tt(const ProjectionStack& proj, std::span<const ViewGeometry> views,
                                 const VolumeGeometry& vol_geom, TTAmplitude amp) {
    if (proj.n_views != int(views.size()))
        throw std::invalid_argument("projection stack does not match views");
    AttenuationVolume out = AttenuationVolume::zeros(vol_geom);
    Lease ctx = scene(vol_geom, proj.det, views);
    const cvpb_tt_options o{int(amp)};
    check(cvpb_group_backproject_tt_host(ctx.group(), &o, proj.values.data(), out.values.data()));
    return out;
}

LinearOperatorPair cvp_pair(const VolumeGeometry& vol, const DetectorGeometry& det,
                            std::span<const ViewGeometry> views, const CvpOptions& opts) {
    auto vs = std::make_shared<std::vector<ViewGeometry>>(views.begin(), views.end());
    LinearOperatorPair p;
    p.vol_geom = vol;
    p.det = det;
    p.n_views = int(vs->size());
    p.forward = [vs, det, opts](const AttenuationVolume& x, ProjectionStack& out) {
        project_cvp_into(x, *vs, det, opts, {}, out);
    };
    p.adjoint = [vs, vol, opts](const ProjectionStack& b, AttenuationVolume& out) {
        backproject_cvp_into(b, *vs, vol, opts, {}, out);
    };
    return p;
}

LinearOperatorPair siddon_pair(const VolumeGeometry& vol, const DetectorGeometry& det,
                               std::span<const ViewGeometry> views, int k_per_edge) {
    auto vs = std::make_shared<std::vector<ViewGeometry>>(views.begin(), views.end());
    LinearOperatorPair p;
    p.vol_geom = vol;
    p.det = det;
    p.n_views = int(vs->size());
    p.forward = [vs, det, k_per_edge](const AttenuationVolume& x, ProjectionStack& out) {
        project_siddon_k_into(x, *vs, det, k_per_edge, {}, out);
    };
    p.adjoint = [vs, vol, k_per_edge](const ProjectionStack& b, AttenuationVolume& out) {
        backproject_siddon_k_into(b, *vs, vol, k_per_edge, {}, out);
    };
    return p;
}

CglsResult cgls_device(const VolumeGeometry& vol, const DetectorGeometry& det,
                       std::span<const ViewGeometry> views, const CvpOptions& opts,
                       const ProjectionStack& b, int iterations) {
    if (iterations < 1) throw std::invalid_argument("cgls needs at least one iteration");
    if (b.det != det || b.n_views != int(views.size()))
        throw std::invalid_argument("cgls data does not match the operator range");
    Lease ctx = scene(vol, det, views);
    const cvpb_cvp_options o = to_c(opts);
    CglsResult res;
    res.x = AttenuationVolume::zeros(vol);
    res.residual_norms.assign(iterations + 1, 0.0);
    check(cvpb_group_cgls_host(ctx.group(), 0, &o, nullptr, nullptr, 1, b.values.data(),
                               res.x.values.data(), iterations, res.residual_norms.data()));
    return res;
}

}  // namespace b200

}  // namespace cbct
