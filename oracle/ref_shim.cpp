// ORACLE TEST INFRASTRUCTURE — not product code.
//
// extern "C" shim around the UNMODIFIED reference library (cbctproj,
// /root/reference/proj/src/*.cpp), compiled from the sources where they lie by
// oracle/Makefile into oracle/_ref/libcbct_ref.so. Only tests/, the smoke
// check in __graft_entry__.py and bench.py's CPU-baseline leg may load it.
//
// Views cross this shim as 17 doubles (the cvpb_view layout of
// include/cvpb200.h): source[3], frame rows e_u,e_v,e_w [9], focal length,
// principal point [2], pixel size [2]; they are rebuilt with the reference's
// own ViewGeometry::make (geometry.cpp:52-88) so both sides of a parity test
// see bit-identical view parameters.
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cbct/cvp.hpp"
#include "cbct/den.hpp"
#include "cbct/geometry.hpp"
#include "cbct/siddon.hpp"
#include "cbct/solver.hpp"

using namespace cbct;

namespace {

thread_local std::string g_err;

enum Status { kOk = 0, kInvalidArgument = 1, kRuntimeError = 2, kOutOfRange = 3, kDomainError = 4, kOther = 5 };

template <class F> int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return kInvalidArgument;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return kOutOfRange;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return kDomainError;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return kRuntimeError;
    } catch (const std::exception& e) {
        g_err = e.what();
        return kOther;
    }
}

ViewGeometry view_from(const double* p) {
    Mat3d fr;
    for (int i = 0; i < 9; ++i) fr.m[i] = p[3 + i];
    return ViewGeometry::make({p[0], p[1], p[2]}, fr, p[12], {p[13], p[14]}, {p[15], p[16]});
}

void view_to(const ViewGeometry& v, double* p) {
    p[0] = v.source().x;
    p[1] = v.source().y;
    p[2] = v.source().z;
    for (int i = 0; i < 9; ++i) p[3 + i] = v.frame().m[i];
    p[12] = v.focal_length();
    p[13] = v.principal_point().x;
    p[14] = v.principal_point().y;
    p[15] = v.pixel_size().x;
    p[16] = v.pixel_size().y;
}

std::vector<ViewGeometry> views_from(const double* p, int n) {
    std::vector<ViewGeometry> v;
    v.reserve(n);
    for (int i = 0; i < n; ++i) v.push_back(view_from(p + 17 * i));
    return v;
}

VolumeGeometry vg_from(const int* counts, const double* voxel) {
    return VolumeGeometry::make({counts[0], counts[1], counts[2]}, {voxel[0], voxel[1], voxel[2]});
}

CvpOptions opts_from(const int* o) {
    CvpOptions c;
    c.scaling = o[0] ? PixelScaling::Exact : PixelScaling::Cos;
    c.elevation_correction = o[1] != 0;
    c.precision = o[2] ? CvpPrecision::Single : CvpPrecision::Double;
    c.r_estimate = o[3] ? RadiusEstimate::CutCentroid : RadiusEstimate::VoxelCenter;
    return c;
}

ExecPolicy exec_from(const int* e) {
    ExecPolicy x;
    if (e) {
        x.threads = e[0];
        x.deterministic = e[1] != 0;
        x.allow_expensive = e[2] != 0;
    }
    return x;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_make_circular_trajectory(double sid, double sdd, int n_views, double arc_deg, int rows,
                                 int cols, double pw, double ph, double* out17) {
    return guarded([&] {
        auto det = DetectorGeometry::make(rows, cols, pw, ph);
        auto views = make_circular_trajectory(sid, sdd, n_views, arc_deg, det);
        for (int v = 0; v < n_views; ++v) view_to(views[v], out17 + 17 * v);
    });
}

int ref_view_standard_matrix(const double* view17, double* P12) {
    return guarded([&] {
        auto P = view_from(view17).standard_matrix();
        std::memcpy(P12, P.data(), sizeof(double) * 12);
    });
}

int ref_view_from_standard_matrix(const double* P12, double pw, double ph, double* out17) {
    return guarded([&] {
        std::array<double, 12> P;
        std::memcpy(P.data(), P12, sizeof(double) * 12);
        view_to(ViewGeometry::from_standard_matrix(P, {pw, ph}), out17);
    });
}

int ref_project_point(const double* view17, const double* x, double* chi) {
    return guarded([&] {
        Vec2d c = view_from(view17).project_point({x[0], x[1], x[2]});
        chi[0] = c.x;
        chi[1] = c.y;
    });
}

int ref_pixel_scale(const double* view17, int rows, int cols, double pw, double ph, int exact,
                    int m, int n, double* out) {
    return guarded([&] {
        auto det = DetectorGeometry::make(rows, cols, pw, ph);
        auto v = view_from(view17);
        *out = exact ? pixel_scale_exact(v, det, m, n) : pixel_scale_cos(v, det, m, n);
    });
}

int ref_project_cvp(const int* counts, const double* voxel, int rows, int cols, double pw,
                    double ph, int n_views, const double* views17, const int* opts4,
                    const int* exec3, const double* vol, double* out, double* view_seconds) {
    return guarded([&] {
        auto vg = vg_from(counts, voxel);
        auto det = DetectorGeometry::make(rows, cols, pw, ph);
        auto views = views_from(views17, n_views);
        AttenuationVolume x{vg, std::vector<double>(vol, vol + vg.voxel_count())};
        ProjectionStack p = ProjectionStack::zeros(det, n_views);
        std::vector<double> vs;
        project_cvp_into(x, views, det, opts_from(opts4), exec_from(exec3), p,
                         view_seconds ? &vs : nullptr);
        std::memcpy(out, p.values.data(), sizeof(double) * p.values.size());
        if (view_seconds) std::memcpy(view_seconds, vs.data(), sizeof(double) * vs.size());
    });
}

int ref_backproject_cvp(const int* counts, const double* voxel, int rows, int cols, double pw,
                        double ph, int n_views, const double* views17, const int* opts4,
                        const int* exec3, const double* proj, double* out, double* view_seconds) {
    return guarded([&] {
        auto vg = vg_from(counts, voxel);
        auto det = DetectorGeometry::make(rows, cols, pw, ph);
        auto views = views_from(views17, n_views);
        ProjectionStack b{det, n_views,
                          std::vector<double>(proj, proj + det.pixel_count() * size_t(n_views))};
        AttenuationVolume x = AttenuationVolume::zeros(vg);
        std::vector<double> vs;
        backproject_cvp_into(b, views, vg, opts_from(opts4), exec_from(exec3), x,
                             view_seconds ? &vs : nullptr);
        std::memcpy(out, x.values.data(), sizeof(double) * x.values.size());
        if (view_seconds) std::memcpy(view_seconds, vs.data(), sizeof(double) * vs.size());
    });
}

// Cut records of voxel (i,j,k): returns the record count in *n_out; writes at
// most cap records (row, column, volume, inv_r2).
int ref_collect_cut_records(const int* counts, const double* voxel, const double* view17, int rows,
                            int cols, double pw, double ph, const int* opts4, int i, int j, int k,
                            int cap, int* rows_out, int* cols_out, double* vol_out,
                            double* invr2_out, int* n_out) {
    return guarded([&] {
        auto vg = vg_from(counts, voxel);
        auto det = DetectorGeometry::make(rows, cols, pw, ph);
        auto recs = collect_cut_records(vg, view_from(view17), det, opts_from(opts4), i, j, k);
        *n_out = int(recs.size());
        for (int r = 0; r < int(recs.size()) && r < cap; ++r) {
            rows_out[r] = recs[r].row;
            cols_out[r] = recs[r].column;
            vol_out[r] = recs[r].volume;
            invr2_out[r] = recs[r].inv_r2;
        }
    });
}

int ref_project_siddon(const int* counts, const double* voxel, int rows, int cols, double pw,
                       double ph, int n_views, const double* views17, int k_per_edge,
                       const int* roi4, const int* exec3, const double* vol, double* out) {
    return guarded([&] {
        auto vg = vg_from(counts, voxel);
        auto det = DetectorGeometry::make(rows, cols, pw, ph);
        auto views = views_from(views17, n_views);
        AttenuationVolume x{vg, std::vector<double>(vol, vol + vg.voxel_count())};
        ProjectionStack p = ProjectionStack::zeros(det, n_views);
        PixelRoi roi;
        if (roi4) roi = {roi4[0], roi4[1], roi4[2], roi4[3]};
        project_siddon_k_into(x, views, det, k_per_edge, exec_from(exec3), p, roi);
        std::memcpy(out, p.values.data(), sizeof(double) * p.values.size());
    });
}

int ref_backproject_siddon(const int* counts, const double* voxel, int rows, int cols, double pw,
                           double ph, int n_views, const double* views17, int k_per_edge,
                           const int* exec3, const double* proj, double* out) {
    return guarded([&] {
        auto vg = vg_from(counts, voxel);
        auto det = DetectorGeometry::make(rows, cols, pw, ph);
        auto views = views_from(views17, n_views);
        ProjectionStack b{det, n_views,
                          std::vector<double>(proj, proj + det.pixel_count() * size_t(n_views))};
        AttenuationVolume x = AttenuationVolume::zeros(vg);
        backproject_siddon_k_into(b, views, vg, k_per_edge, exec_from(exec3), x);
        std::memcpy(out, x.values.data(), sizeof(double) * x.values.size());
    });
}

// trace_ray: writes up to cap (i,j,k,length) tuples, count in *n_out.
int ref_trace_ray(const int* counts, const double* voxel, const double* src, const double* tgt,
                  int cap, int* ijk_out, double* len_out, int* n_out) {
    return guarded([&] {
        auto vg = vg_from(counts, voxel);
        auto list = trace_ray(vg, {src[0], src[1], src[2]}, {tgt[0], tgt[1], tgt[2]});
        *n_out = int(list.size());
        for (int r = 0; r < int(list.size()) && r < cap; ++r) {
            ijk_out[3 * r] = list[r].i;
            ijk_out[3 * r + 1] = list[r].j;
            ijk_out[3 * r + 2] = list[r].k;
            len_out[r] = list[r].length;
        }
    });
}

int ref_fill_uniform01(double* out, std::size_t n, std::uint64_t seed) {
    return guarded([&] { fill_uniform01(std::span<double>(out, n), seed); });
}

namespace {
LinearOperatorPair make_pair(const int* counts, const double* voxel, int rows, int cols, double pw,
                             double ph, int n_views, const double* views17, int projector,
                             const int* opts4, int k_per_edge) {
    auto vg = vg_from(counts, voxel);
    auto det = DetectorGeometry::make(rows, cols, pw, ph);
    auto views = std::make_shared<std::vector<ViewGeometry>>(views_from(views17, n_views));
    LinearOperatorPair p;
    p.vol_geom = vg;
    p.det = det;
    p.n_views = n_views;
    if (projector == 0) {
        CvpOptions o = opts_from(opts4);
        p.forward = [views, det, o](const AttenuationVolume& x, ProjectionStack& out) {
            project_cvp_into(x, *views, det, o, {}, out);
        };
        p.adjoint = [views, vg, o](const ProjectionStack& b, AttenuationVolume& out) {
            backproject_cvp_into(b, *views, vg, o, {}, out);
        };
    } else {
        p.forward = [views, det, k_per_edge](const AttenuationVolume& x, ProjectionStack& out) {
            project_siddon_k_into(x, *views, det, k_per_edge, {}, out);
        };
        p.adjoint = [views, vg, k_per_edge](const ProjectionStack& b, AttenuationVolume& out) {
            backproject_siddon_k_into(b, *views, vg, k_per_edge, {}, out);
        };
    }
    return p;
}
} // namespace

// projector: 0 = CVP (opts4), 1 = Siddon-K (k_per_edge).
int ref_adjoint_test(const int* counts, const double* voxel, int rows, int cols, double pw,
                     double ph, int n_views, const double* views17, int projector,
                     const int* opts4, int k_per_edge, std::uint64_t seed, double* out) {
    return guarded([&] {
        *out = adjoint_test(
            make_pair(counts, voxel, rows, cols, pw, ph, n_views, views17, projector, opts4, k_per_edge),
            seed);
    });
}

int ref_cgls(const int* counts, const double* voxel, int rows, int cols, double pw, double ph,
             int n_views, const double* views17, int projector, const int* opts4, int k_per_edge,
             const double* b, int iterations, double* x_out, double* residuals_out) {
    return guarded([&] {
        auto pair = make_pair(counts, voxel, rows, cols, pw, ph, n_views, views17, projector, opts4,
                              k_per_edge);
        ProjectionStack bs{pair.det, n_views,
                           std::vector<double>(b, b + pair.range_size())};
        CglsResult r = cgls(pair, bs, iterations);
        std::memcpy(x_out, r.x.values.data(), sizeof(double) * r.x.values.size());
        std::memcpy(residuals_out, r.residual_norms.data(),
                    sizeof(double) * r.residual_norms.size());
    });
}

// DEN I/O (den.cpp:27-100): write (y, x, z, float32 payload) / read back.
int ref_den_write(const char* path, int y, int x, int z, const float* values) {
    return guarded([&] {
        DenFile d;
        d.dim_y = std::uint16_t(y);
        d.dim_x = std::uint16_t(x);
        d.dim_z = std::uint16_t(z);
        d.values.assign(values, values + d.value_count());
        den_write(path, d);
    });
}

// dims_out[3] = (y, x, z); copies at most cap values
int ref_den_read(const char* path, int* dims_out, float* values, std::size_t cap) {
    return guarded([&] {
        DenFile d = den_read(path);
        dims_out[0] = d.dim_y;
        dims_out[1] = d.dim_x;
        dims_out[2] = d.dim_z;
        std::memcpy(values, d.values.data(), sizeof(float) * std::min(cap, d.values.size()));
    });
}

// volume -> DEN -> file (to_den of an AttenuationVolume, float64 -> float32)
int ref_den_write_volume(const char* path, const int* counts, const double* voxel,
                         const double* values) {
    return guarded([&] {
        auto g = VolumeGeometry::make({counts[0], counts[1], counts[2]}, {voxel[0], voxel[1], voxel[2]});
        AttenuationVolume v{g, std::vector<double>(values, values + g.voxel_count())};
        den_write(path, to_den(v));
    });
}

} // extern "C"
