// Host-side CVP introspection helpers of the drop-in API (float64):
// column_cuts, row_breakpoints, elevation_corrected_split (reference
// cvp.hpp:48-79, cvp.cpp:506-568). They expose the geometry of one voxel
// column / one cut as polygons and row segments — the bookkeeping the
// reference's unit tests pin (test_cvp.cpp:69-317). The projector itself never
// materialises these: the device kernels integrate the same quantities in
// registers (csrc/cvp_device.cuh). Semantics follow the reference functions
// cited per block; the code is this library's own.
#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <vector>

#include "cbct_b200/cbct.hpp"

namespace cbct {

namespace {

// Horizontal reduction of a view (ViewCtx, cvp.cpp:26-70): the camera rows
// r0, r2 restricted to x1x2, the source, and the chi2 <-> z maps at a depth.
struct Planar {
    Vec2d w1, w3, s;
    double s3, pp2, f_b2, b2_f;

    explicit Planar(const ViewGeometry& v) {
        const Mat3d& C = v.camera_matrix();
        w1 = {C(0, 0), C(0, 1)};
        w3 = {C(2, 0), C(2, 1)};
        s = v.source().xy();
        s3 = v.source().z;
        pp2 = v.principal_point().y;
        f_b2 = v.focal_length() / v.pixel_size().y;
        b2_f = v.pixel_size().y / v.focal_length();
    }
    double depth(Vec2d p) const { return dot(w3, p - s); }
    double chi1(Vec2d p) const { return dot(w1, p - s) / depth(p); }
    double z_at(double chi2, double d) const { return s3 + (pp2 - chi2) * b2_f * d; }
    double chi2_at(double z, double d) const { return pp2 - (z - s3) * f_b2 / d; }
    // pre-image of chi1 <= c: the half-plane (w1 - c w3).(p - s) <= 0
    HalfPlane2D chi1_at_most(double c) const {
        const Vec2d nrm = w1 - c * w3;
        return HalfPlane2D::from_line(nrm, dot(nrm, s));
    }
};

// Column range n_lo..n_hi of a base polygon (BandCutter, cvp.cpp:73-98).
void column_range(const Planar& P, const Polygon2D& base, int& n_lo, int& n_hi) {
    double lo = std::numeric_limits<double>::infinity(), hi = -lo;
    for (int i = 0; i < base.size(); ++i) {
        if (!(P.depth(base[i]) > 0.0))
            throw std::runtime_error("numerical degeneracy: voxel base reaches the source plane");
        const double c = P.chi1(base[i]);
        lo = std::min(lo, c);
        hi = std::max(hi, c);
    }
    n_lo = int(std::ceil(lo - 0.5));
    n_hi = int(std::floor(hi + 0.5));
}

// What the row split needs of one cut (CutInfo / fill_cut_info, cvp.cpp:101-136).
struct Cut {
    double d0 = 0.0, hw = 0.0, halfw = 0.0;
};

Cut describe(const Planar& P, const Polygon2D& piece, bool need_width) {
    const double A = area(piece);
    const Vec2d rel = centroid(piece) - P.s;
    const double rho = std::sqrt(dot(rel, rel));
    Cut c;
    c.d0 = dot(P.w3, rel);
    c.hw = c.d0 / rho;
    if (need_width) {
        // extent of the piece across the horizontal source direction; the
        // rectangle's half-width is half of area / extent
        const Vec2d across = perp(rel) / rho;
        double lo = std::numeric_limits<double>::infinity(), hi = -lo;
        for (int i = 0; i < piece.size(); ++i) {
            const double t = dot(across, piece[i]);
            lo = std::min(lo, t);
            hi = std::max(hi, t);
        }
        if (hi - lo > 0.0) c.halfw = A / (hi - lo) * 0.5;
    }
    return c;
}

// Exact mean of clamp(alpha + beta xi, z_lo, z_hi) over xi in [-w, w]
// (clamp_mean, cvp.cpp:161-175): the clamped ramp integrated piecewise.
double ramp_mean(double alpha, double beta, double w, double z_lo, double z_hi) {
    const double s = std::abs(beta) * w;
    if (!(s > 0.0)) return std::clamp(alpha, z_lo, z_hi);
    const double a = alpha - s, b = alpha + s;
    if (a >= z_lo && b <= z_hi) return alpha;
    if (b <= z_lo) return z_lo;
    if (a >= z_hi) return z_hi;
    const double ca = std::clamp(a, z_lo, z_hi), cb = std::clamp(b, z_lo, z_hi);
    const double under = std::max(0.0, std::min(b, z_lo) - a);
    const double over = std::max(0.0, b - std::max(a, z_hi));
    return (z_lo * under + (cb * cb - ca * ca) / 2.0 + z_hi * over) / (b - a);
}

// Rows of one cut over [z_lo, z_hi] with their z shares (visit_rows,
// cvp.cpp:180-235, unclamped rows, unit area): shares are differences of the
// clamped (or ramp-averaged) z at consecutive row boundaries, so they
// telescope to z_hi - z_lo.
std::vector<RowSegment> split_rows(const Planar& P, const Cut& c, double z_lo, double z_hi, bool corrected) {
    const double dd = corrected ? std::abs(c.hw) * c.halfw : 0.0;
    double lo = std::numeric_limits<double>::infinity(), hi = -lo;
    for (double z : {z_lo, z_hi})
        for (double d : {c.d0 - dd, c.d0 + dd}) {
            const double chi = P.chi2_at(z, d);
            lo = std::min(lo, chi);
            hi = std::max(hi, chi);
        }
    const int first = int(std::ceil(lo - 0.5)), last = int(std::floor(hi + 0.5));
    std::vector<RowSegment> out;
    if (first > last) return out;
    auto boundary_z = [&](double chi) {
        const double alpha = P.z_at(chi, c.d0);
        if (!corrected) return std::clamp(alpha, z_lo, z_hi);
        return ramp_mean(alpha, (P.pp2 - chi) * P.b2_f * c.hw, c.halfw, z_lo, z_hi);
    };
    double upper = boundary_z(double(first) - 0.5);
    for (int m = first; m <= last; ++m) {
        const double lower = boundary_z(double(m) + 0.5);
        if (upper - lower > 0.0) out.push_back({m, upper - lower});
        upper = lower;
    }
    return out;
}

}  // namespace

// column_cuts (cvp.cpp:506-520): one piece per detector column between the
// pre-images of chi1 = n -+ 1/2, columns outside the detector included.
std::vector<ColumnCut> column_cuts(const ViewGeometry& view, const DetectorGeometry& det,
                                   const Polygon2D& voxel_base) {
    (void)det;
    if (voxel_base.size() < 3) throw std::invalid_argument("voxel base polygon is degenerate");
    const Planar P(view);
    int n_lo, n_hi;
    column_range(P, voxel_base, n_lo, n_hi);
    std::vector<ColumnCut> cuts;
    for (int n = n_lo; n <= n_hi; ++n) {
        const Polygon2D piece = n_lo == n_hi ? voxel_base
                                             : band_cut(voxel_base, P.chi1_at_most(n - 0.5),
                                                        P.chi1_at_most(n + 0.5));
        if (piece.empty()) continue;
        const double A = area(piece);
        if (A > 0.0) cuts.push_back({n, piece, A, centroid(piece)});
    }
    return cuts;
}

// row_breakpoints (cvp.cpp:522-548): the plain split of the vertical segment
// [z_lo, z_hi] above one base-plane point; empty when it misses the detector.
std::vector<RowSegment> row_breakpoints(const ViewGeometry& view, const DetectorGeometry& det,
                                        const Vec2d& centroid_xy, double z_lo, double z_hi) {
    if (!(z_hi > z_lo)) return {};
    const Planar P(view);
    const double d0 = P.depth(centroid_xy);
    if (!(d0 > 0.0)) return {};
    const double c1 = P.chi1(centroid_xy);
    if (c1 < -0.5 || c1 > det.cols - 0.5) return {};
    if (P.chi2_at(z_lo, d0) < -0.5 || P.chi2_at(z_hi, d0) > det.rows - 0.5) return {};
    Cut c;
    c.d0 = d0;
    return split_rows(P, c, z_lo, z_hi, false);
}

// elevation_corrected_split (cvp.cpp:550-568): the split with the cut modelled
// as a +-halfw rectangle in the source plane through its centroid.
std::vector<RowSegment> elevation_corrected_split(const ViewGeometry& view, const DetectorGeometry& det,
                                                  const ColumnCut& cut, double z_lo, double z_hi,
                                                  double elevation) {
    (void)det;
    if (!(z_hi > z_lo)) return {};
    if (cut.polygon.size() < 3 || !(cut.area > 0.0)) throw std::invalid_argument("degenerate column cut");
    const Planar P(view);
    const Cut c = describe(P, cut.polygon, true);
    if (!(c.d0 > 0.0)) return {};
    return split_rows(P, c, z_lo, z_hi, elevation > 0.0 && c.halfw > 0.0);
}

}  // namespace cbct
