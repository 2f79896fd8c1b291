// Reference-style unit checks compiled against the drop-in headers
// (include/cbct/*.hpp -> include/cbct_b200/cbct.hpp) and linked to
// libcbct_b200.so: the same calls a reference caller makes
// (tests/test_cvp.cpp, test_siddon.cpp, test_geometry.cpp, test_solver.cpp of
// the reference), now served by the GPU. Device arithmetic is float32, so
// exactness checks use float32 tolerances (stated per check).
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>

#include "cbct/cvp.hpp"
#include "cbct/siddon.hpp"
#include "cbct/solver.hpp"

using namespace cbct;

static int g_fail = 0, g_pass = 0;

#define CHECK(cond)                                                        \
    do {                                                                   \
        if (cond) {                                                        \
            ++g_pass;                                                      \
        } else {                                                           \
            ++g_fail;                                                      \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);    \
        }                                                                  \
    } while (0)

template <class E, class F> bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void fill_random(std::vector<double>& v, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    for (double& x : v) x = uniform01(rng);
}

static void test_geometry() {
    auto det = DetectorGeometry::make(128, 128, 1.0, 1.0);
    auto views = make_circular_trajectory(541.0, 949.0, 720, 360.0, det);
    CHECK(views.size() == 720);
    CHECK(std::abs(views[1].source().x - 541.0 * std::cos(0.5 * M_PI / 180.0)) < 1e-12);
    CHECK(throws<std::invalid_argument>([&] { make_circular_trajectory(541, 949, 0, 360, det); }));
    Mat3d good = Mat3d::from_rows({0, 1, 0}, {0, 0, -1}, {-1, 0, 0});
    Mat3d flipped = Mat3d::from_rows({0, -1, 0}, {0, 0, 1}, {-1, 0, 0});
    CHECK(!throws<std::exception>([&] { ViewGeometry::make({541, 0, 0}, good, 949.0, {63.5, 63.5}, {1, 1}); }));
    CHECK(throws<std::invalid_argument>([&] { ViewGeometry::make({541, 0, 0}, flipped, 949.0, {63.5, 63.5}, {1, 1}); }));
    auto v = make_circular_trajectory(541.0, 949.0, 5, 360.0, det)[0];
    Vec2d c = v.project_point({0, 0, 0});
    CHECK(std::abs(c.x - 63.5) < 1e-12 && std::abs(c.y - 63.5) < 1e-12);
    CHECK(throws<std::domain_error>([&] { (void)v.project_point({1000.0, 0.0, 0.0}); }));
    auto P = v.standard_matrix();
    auto back = ViewGeometry::from_standard_matrix(P, det.pixel_size());
    CHECK(norm(back.source() - v.source()) < 1e-9);
}

static void test_cvp() {
    auto geom = VolumeGeometry::make({16, 16, 16}, {1.0, 1.0, 1.0});
    auto det = DetectorGeometry::make(32, 32, 1.0, 1.0);
    auto views = make_circular_trajectory(40.0, 70.0, 8, 360.0, det);

    // zeros and linearity (test_cvp.cpp:319-335), linearity to float32 rounding
    auto zero = project_cvp(AttenuationVolume::zeros(geom), views, det);
    bool allz = true;
    for (double p : zero.values) allz &= (p == 0.0);
    CHECK(allz);
    auto x = AttenuationVolume::zeros(geom);
    fill_random(x.values, 3);
    auto dx = x;
    for (double& t : dx.values) t *= 2.0;
    auto p1 = project_cvp(x, views, det), p2 = project_cvp(dx, views, det);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < p1.values.size(); ++i) {
        num += (p2.values[i] - 2 * p1.values[i]) * (p2.values[i] - 2 * p1.values[i]);
        den += p2.values[i] * p2.values[i];
    }
    CHECK(std::sqrt(num / den) < 1e-6);

    // unsupported configurations (test_cvp.cpp:337-347)
    auto inside = make_circular_trajectory(4.0, 70.0, 1, 360.0, det);
    CHECK(throws<std::runtime_error>([&] { project_cvp(AttenuationVolume::zeros(geom), inside, det); }));
    auto other = DetectorGeometry::make(32, 32, 0.5, 1.0);
    CHECK(throws<std::invalid_argument>([&] { project_cvp(AttenuationVolume::zeros(geom), views, other); }));

    // adjoint identity for every option combination (test_cvp.cpp:349-373; float32 bar)
    int combo = 0;
    for (auto scaling : {PixelScaling::Cos, PixelScaling::Exact})
        for (bool elev : {false, true})
            for (auto rest : {RadiusEstimate::VoxelCenter, RadiusEstimate::CutCentroid}) {
                CvpOptions opts{scaling, elev, CvpPrecision::Double, rest};
                auto xx = AttenuationVolume::zeros(geom);
                auto b = ProjectionStack::zeros(det, int(views.size()));
                fill_random(xx.values, 400 + combo);
                fill_random(b.values, 500 + combo);
                ++combo;
                auto ax = project_cvp(xx, views, det, opts);
                auto atb = backproject_cvp(b, views, geom, opts);
                double lhs = 0, rhs = 0;
                for (std::size_t i = 0; i < b.values.size(); ++i) lhs += b.values[i] * ax.values[i];
                for (std::size_t i = 0; i < xx.values.size(); ++i) rhs += xx.values[i] * atb.values[i];
                CHECK(std::abs(lhs - rhs) <= 1e-5 * std::max(std::abs(lhs), std::abs(rhs)));
            }
    CHECK(combo == 8);

    // single-pixel impulse = forward bookkeeping x scale (test_cvp.cpp:375-408)
    {
        auto g8 = VolumeGeometry::make({8, 8, 8}, {1.0, 1.0, 1.0});
        auto d24 = DetectorGeometry::make(24, 24, 1.0, 1.0);
        auto v1 = make_circular_trajectory(30.0, 50.0, 1, 360.0, d24);
        CvpOptions opts{};
        auto central = collect_cut_records(g8, v1[0], d24, opts, 4, 4, 4);
        CHECK(!central.empty());
        auto best = central[0];
        for (const auto& r : central)
            if (r.volume > best.volume) best = r;
        auto proj = ProjectionStack::zeros(d24, 1);
        proj.at(0, best.row, best.column) = 1.0;
        auto vol = backproject_cvp(proj, v1, g8, opts);
        const double scale = pixel_scale_exact(v1[0], d24, best.row, best.column);
        double worst = 0, peak = 0;
        for (int k = 0; k < 8; ++k)
            for (int j = 0; j < 8; ++j)
                for (int i = 0; i < 8; ++i) {
                    double want = 0;
                    for (const auto& rec : collect_cut_records(g8, v1[0], d24, opts, i, j, k))
                        if (rec.row == best.row && rec.column == best.column)
                            want += rec.volume * rec.inv_r2 * scale;
                    worst = std::max(worst, std::abs(vol.at(i, j, k) - want));
                    peak = std::max(peak, std::abs(want));
                }
        CHECK(worst <= 1e-5 * peak);
    }

    // cut records conserve the voxel volume (test_cvp.cpp:410-432; float32 areas)
    {
        auto g64 = VolumeGeometry::make({64, 64, 64}, {0.5, 0.5, 0.5});
        auto desk = DetectorGeometry::make(128, 128, 1.0, 1.0);
        auto vv = make_circular_trajectory(541.0, 949.0, 36, 360.0, desk);
        std::mt19937_64 rng(17);
        for (int t = 0; t < 20; ++t) {
            int i = int(rng() % 64), j = int(rng() % 64), k = int(rng() % 64);
            const auto& view = vv[rng() % vv.size()];
            for (bool elev : {false, true}) {
                CvpOptions o{PixelScaling::Exact, elev, CvpPrecision::Double, RadiusEstimate::CutCentroid};
                double sum = 0;
                for (const auto& r : collect_cut_records(g64, view, desk, o, i, j, k)) sum += r.volume;
                CHECK(std::abs(sum - 0.125) < 1e-6);
            }
        }
    }

    // single precision tracks double precision (test_cvp.cpp:434-458)
    {
        auto g64 = VolumeGeometry::make({64, 64, 64}, {0.5, 0.5, 0.5});
        auto vol = AttenuationVolume::zeros(g64);
        fill_random(vol.values, 9);
        auto desk = DetectorGeometry::make(128, 128, 1.0, 1.0);
        auto vv = make_circular_trajectory(541.0, 949.0, 6, 360.0, desk);
        CvpOptions so;
        so.precision = CvpPrecision::Single;
        auto pd = project_cvp(vol, vv, desk), ps = project_cvp(vol, vv, desk, so);
        for (int v = 0; v < pd.n_views; ++v)
            CHECK(relative_projector_error(ps.view(v), pd.view(v)) < 1e-1);  // percent: < 1e-3 relative
    }
}

static void test_siddon() {
    auto vol = VolumeGeometry::make({4, 4, 4}, {1.0, 1.0, 1.0});
    // axis-aligned ray through row j=1, k=2 (test_siddon.cpp:31-80)
    auto list = trace_ray(vol, {-10.0, -0.5, 0.5}, {10.0, -0.5, 0.5});
    CHECK(list.size() == 4);
    double total = 0;
    for (const auto& r : list) total += r.length;
    CHECK(std::abs(total - 4.0) < 1e-12);
    auto diag = trace_ray(VolumeGeometry::make({1, 1, 1}, {1.0, 1.0, 1.0}), {-1, -1, -1}, {1, 1, 1});
    CHECK(diag.size() == 1 && std::abs(diag[0].length - std::sqrt(3.0)) < 1e-12);
    CHECK(trace_ray(vol, {-10.0, 50.0, 0.0}, {10.0, 50.0, 0.0}).empty());

    auto geom = VolumeGeometry::make({16, 16, 16}, {1.0, 1.0, 1.0});
    auto det = DetectorGeometry::make(32, 32, 1.0, 1.0);
    auto views = make_circular_trajectory(40.0, 70.0, 4, 360.0, det);
    auto x = AttenuationVolume::zeros(geom);
    CHECK(throws<std::invalid_argument>([&] { project_siddon_k(x, views, det, 128); }));
    fill_random(x.values, 5);
    auto b = ProjectionStack::zeros(det, 4);
    fill_random(b.values, 6);
    for (int K : {1, 2}) {
        auto ax = project_siddon_k(x, views, det, K);
        auto atb = backproject_siddon_k(b, views, geom, K);
        double lhs = 0, rhs = 0;
        for (std::size_t i = 0; i < b.values.size(); ++i) lhs += b.values[i] * ax.values[i];
        for (std::size_t i = 0; i < x.values.size(); ++i) rhs += x.values[i] * atb.values[i];
        CHECK(std::abs(lhs - rhs) <= 1e-5 * std::abs(lhs));
    }
}

static void test_solver() {
    auto geom = VolumeGeometry::make({16, 16, 16}, {1.0, 1.0, 1.0});
    auto det = DetectorGeometry::make(32, 32, 1.0, 1.0);
    auto views = make_circular_trajectory(40.0, 70.0, 60, 360.0, det);
    auto pair = b200::cvp_pair(geom, det, views);
    auto x_true = AttenuationVolume::zeros(geom);
    for (int k = 0; k < 16; ++k)
        for (int j = 0; j < 16; ++j)
            for (int i = 0; i < 16; ++i) {
                double r2 = (i - 7.5) * (i - 7.5) + (j - 7.5) * (j - 7.5) + (k - 7.5) * (k - 7.5);
                x_true.at(i, j, k) = std::exp(-r2 / 18.0);
            }
    auto b = ProjectionStack::zeros(det, pair.n_views);
    pair.forward(x_true, b);
    auto res = cgls(pair, b, 40);
    CHECK(res.residual_norms.back() / res.residual_norms[0] < 1e-3);
    auto dev = b200::cgls_device(geom, det, views, {}, b, 40);
    CHECK(dev.residual_norms.back() / dev.residual_norms[0] < 1e-3);
    CHECK(std::abs(dev.residual_norms[5] / res.residual_norms[5] - 1.0) < 1e-4);
    CHECK(adjoint_test(pair, 1) < 1e-5);
    CHECK(adjoint_test(b200::siddon_pair(geom, det, views, 2), 1) < 1e-5);
    auto tt = b200::project_tt(x_true, views, det);
    CHECK(tt.values.size() == b.values.size());
}

int main() {
    test_geometry();
    test_cvp();
    test_siddon();
    test_solver();
    std::printf("DROPIN %s: %d checks passed, %d failed\n", g_fail ? "FAIL" : "PASS", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
