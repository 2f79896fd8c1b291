// cbct_b200 — convex polygon kernel of the drop-in API.
//
// Contract of the reference header cbct/polygon.hpp (polygon.hpp:14-164):
//   * BasicHalfPlane2D<T>  closed half-plane {x : n.x <= c}, unit normal
//     (from_line normalises; a zero normal is std::invalid_argument);
//   * BasicPolygon2D<T>    convex CCW polygon of at most 8 vertices
//     (std::length_error past that), rectangle(lo, hi) factory;
//   * area / centroid      shoelace moments (centroid of a zero-area polygon
//     is std::domain_error);
//   * clip                 one Sutherland–Hodgman pass, vertices on the line
//     kept, near-duplicate vertices (1e-12 of the coordinate scale) merged,
//     fewer than 3 vertices or an area below 1e-14 scale^2 -> empty;
//   * band_cut             clip by `upper`, then by the complement of `lower`.
// The CVP kernels never build polygons (they integrate clipped moments in
// registers, csrc/cvp_device.cuh); this header serves the host-side
// introspection helpers (column_cuts & co.) and reference callers that use
// Polygon2D directly.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <initializer_list>
#include <stdexcept>

#include "cbct_b200/vec.hpp"

namespace cbct {

template <typename T> struct BasicHalfPlane2D {
    Vec2<T> normal{};
    T offset{};

    static BasicHalfPlane2D from_line(Vec2<T> n, T c) {
        const T len = std::sqrt(n.x * n.x + n.y * n.y);
        if (!(len > T(0))) throw std::invalid_argument("half-plane normal must be nonzero");
        return BasicHalfPlane2D{n / len, c / len};
    }
    BasicHalfPlane2D complement() const { return BasicHalfPlane2D{-normal, -offset}; }
    T signed_distance(Vec2<T> p) const { return dot(normal, p) - offset; }
};

template <typename T> class BasicPolygon2D {
  public:
    static constexpr int capacity = 8;

    BasicPolygon2D() = default;
    BasicPolygon2D(std::initializer_list<Vec2<T>> pts) {
        for (const Vec2<T>& p : pts) push_back(p);
    }

    static BasicPolygon2D rectangle(Vec2<T> lo, Vec2<T> hi) {
        if (!(lo.x < hi.x && lo.y < hi.y)) throw std::invalid_argument("rectangle corners must be ordered");
        return BasicPolygon2D{{lo.x, lo.y}, {hi.x, lo.y}, {hi.x, hi.y}, {lo.x, hi.y}};
    }

    int size() const { return count_; }
    bool empty() const { return count_ == 0; }
    Vec2<T> operator[](int i) const { return pts_[i]; }
    void clear() { count_ = 0; }

    void push_back(Vec2<T> p) {
        if (count_ >= capacity) throw std::length_error("polygon capacity exceeded");
        pts_[count_] = p;
        ++count_;
    }

    // largest |coordinate| over the vertices: the length scale of the
    // degeneracy thresholds
    T scale() const {
        T s = T(0);
        for (int i = 0; i < count_; ++i) s = std::max(s, std::max(std::abs(pts_[i].x), std::abs(pts_[i].y)));
        return s;
    }

  private:
    std::array<Vec2<T>, capacity> pts_{};
    int count_ = 0;
};

// (edge sums in vertex order 0->1, 1->2, ..., n-1->0)
template <typename T> T area(const BasicPolygon2D<T>& p) {
    const int n = p.size();
    T twice = T(0);
    for (int i = 0; i < n; ++i) twice += cross(p[i], p[i + 1 < n ? i + 1 : 0]);
    return twice / T(2);
}

template <typename T> Vec2<T> centroid(const BasicPolygon2D<T>& p) {
    const int n = p.size();
    T twice = T(0);
    Vec2<T> m{};
    for (int i = 0; i < n; ++i) {
        const Vec2<T> a = p[i], b = p[i + 1 < n ? i + 1 : 0];
        const T c = cross(a, b);
        twice += c;
        m = m + (a + b) * c;
    }
    if (!(std::abs(twice) > T(0))) throw std::domain_error("centroid of a degenerate polygon");
    return m / (T(3) * twice);
}

namespace poly_detail {

template <typename T> struct Ring {  // one clip's raw output (n + 1 vertices at most)
    std::array<Vec2<T>, 9> v{};
    int n = 0;
    void add(Vec2<T> p) { v[n++] = p; }
};

template <typename T> bool close(Vec2<T> a, Vec2<T> b, T eps) {
    return std::abs(a.x - b.x) <= eps && std::abs(a.y - b.y) <= eps;
}

}  // namespace poly_detail

template <typename T> BasicPolygon2D<T> clip(const BasicPolygon2D<T>& poly, const BasicHalfPlane2D<T>& hp) {
    const int n = poly.size();
    if (n == 0) return {};
    poly_detail::Ring<T> ring;
    // walk edges (i -> i+1); every vertex with d <= 0 is kept as is, and a
    // strict sign change adds the crossing (t measured from the edge start)
    std::array<T, BasicPolygon2D<T>::capacity> d{};
    for (int i = 0; i < n; ++i) d[i] = hp.signed_distance(poly[i]);
    for (int i = 0; i < n; ++i) {
        const int k = i + 1 < n ? i + 1 : 0;
        const Vec2<T> a = poly[i], b = poly[k];
        if (d[i] <= T(0)) ring.add(a);
        const bool crosses = (d[i] < T(0) && d[k] > T(0)) || (d[i] > T(0) && d[k] < T(0));
        if (crosses) ring.add(a + (b - a) * (d[i] / (d[i] - d[k])));
    }
    if (ring.n < 3) return {};
    T eps = T(0);
    for (int i = 0; i < ring.n; ++i) eps = std::max(eps, std::max(std::abs(ring.v[i].x), std::abs(ring.v[i].y)));
    eps *= T(1e-12);
    // drop vertices that repeat their predecessor, then a last vertex that
    // repeats the first
    std::array<Vec2<T>, 9> keep{};
    int m = 0;
    keep[m++] = ring.v[0];
    for (int i = 1; i < ring.n; ++i)
        if (!poly_detail::close(ring.v[i], keep[m - 1], eps)) keep[m++] = ring.v[i];
    if (m >= 2 && poly_detail::close(keep[m - 1], keep[0], eps)) --m;
    if (m < 3) return {};
    BasicPolygon2D<T> out;
    for (int i = 0; i < m; ++i) out.push_back(keep[i]);
    const T s = out.scale();
    if (area(out) < T(1e-14) * s * s) return {};
    return out;
}

template <typename T>
BasicPolygon2D<T> band_cut(const BasicPolygon2D<T>& square, const BasicHalfPlane2D<T>& lower,
                           const BasicHalfPlane2D<T>& upper) {
    const BasicPolygon2D<T> below_upper = clip(square, upper);
    return clip(below_upper, lower.complement());
}

using HalfPlane2D = BasicHalfPlane2D<double>;
using Polygon2D = BasicPolygon2D<double>;

}  // namespace cbct
