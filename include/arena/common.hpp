// arena/common.hpp — drop-in re-declaration of the reference's core types.
//
// API-compatible with /root/reference/proj/include/arena/common.hpp:14-23
// (Vec3 as std::array<double,3>, the four vector helpers, ScalarField as a
// std::function) so code written against the reference compiles unchanged
// against this framework.  Only what the spectral-solve boundary needs.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace arena {

/// A point / vector in the unit cube.
using Vec3 = std::array<double, 3>;

inline double dot(const Vec3& u, const Vec3& v) { return u[0] * v[0] + u[1] * v[1] + u[2] * v[2]; }
inline double norm(const Vec3& v) { return std::sqrt(dot(v, v)); }
inline Vec3 operator+(const Vec3& u, const Vec3& v) { return Vec3{u[0] + v[0], u[1] + v[1], u[2] + v[2]}; }
inline Vec3 operator-(const Vec3& u, const Vec3& v) { return Vec3{u[0] - v[0], u[1] - v[1], u[2] - v[2]}; }
inline Vec3 operator*(double a, const Vec3& v) { return Vec3{a * v[0], a * v[1], a * v[2]}; }

/// Scalar field x -> value, e.g. a source f or an analytic u.
using ScalarField = std::function<double(const Vec3&)>;

}  // namespace arena
