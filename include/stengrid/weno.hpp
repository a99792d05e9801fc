// stengrid/weno.hpp — drop-in for the reference WENO5 advection API
// (/root/reference/proj/include/stengrid/weno.hpp:1-30). weno_advect runs on
// the GPU (csrc/weno.cu), bitwise identical to the reference.
#pragma once

#include "stengrid/grid.hpp"

namespace stengrid {

struct VelocityField {
  Grid2D u;
  Grid2D v;
};

enum class UpwindSide { Left, Right };

inline UpwindSide upwind_side(double velocity) { return velocity < 0.0 ? UpwindSide::Right : UpwindSide::Left; }

/// weno.cpp:13-48 (host scalar helper, same arithmetic as the device kernel).
inline double weno_derivative_7(const double* w7, double invH, UpwindSide side) {
  auto combine = [](double v1, double v2, double v3, double v4, double v5) {
    constexpr double eps = 1e-6;
    const double c1 = v1 * (1.0 / 3.0) - v2 * (7.0 / 6.0) + v3 * (11.0 / 6.0);
    const double c2 = -v2 * (1.0 / 6.0) + v3 * (5.0 / 6.0) + v4 * (1.0 / 3.0);
    const double c3 = v3 * (1.0 / 3.0) + v4 * (5.0 / 6.0) - v5 * (1.0 / 6.0);
    const double d1 = v1 - 2.0 * v2 + v3, d2 = v2 - 2.0 * v3 + v4, d3 = v3 - 2.0 * v4 + v5;
    const double s1 = (13.0 / 12.0) * d1 * d1 + 0.25 * (v1 - 4.0 * v2 + 3.0 * v3) * (v1 - 4.0 * v2 + 3.0 * v3);
    const double s2 = (13.0 / 12.0) * d2 * d2 + 0.25 * (v2 - v4) * (v2 - v4);
    const double s3 = (13.0 / 12.0) * d3 * d3 + 0.25 * (3.0 * v3 - 4.0 * v4 + v5) * (3.0 * v3 - 4.0 * v4 + v5);
    const double a1 = 0.1 / ((eps + s1) * (eps + s1));
    const double a2 = 0.6 / ((eps + s2) * (eps + s2));
    const double a3 = 0.3 / ((eps + s3) * (eps + s3));
    return (a1 * c1 + a2 * c2 + a3 * c3) / (a1 + a2 + a3);
  };
  if (side == UpwindSide::Left)
    return combine((w7[1] - w7[0]) * invH, (w7[2] - w7[1]) * invH, (w7[3] - w7[2]) * invH, (w7[4] - w7[3]) * invH,
                   (w7[5] - w7[4]) * invH);
  return combine((w7[6] - w7[5]) * invH, (w7[5] - w7[4]) * invH, (w7[4] - w7[3]) * invH, (w7[3] - w7[2]) * invH,
                 (w7[2] - w7[1]) * invH);
}

/// weno.cpp:50-94 — -(u dphi/dx + v dphi/dy), WENO5 upwinded, periodic; on the GPU.
inline Grid2D weno_advect(const Grid2D& phi, const VelocityField& vel, int numTiles = 1, int numWorkers = 1) {
  if (!phi.same_shape(vel.u) || !phi.same_shape(vel.v))
    throw std::invalid_argument("weno_advect: velocity shape does not match the field");
  if (phi.nx < 7 || phi.ny < 7) throw std::invalid_argument("weno_advect: need nx, ny >= 7");
  (void)make_tiles(phi.ny, numTiles, Extents{0, 0, 3, 3});
  if (numWorkers < 1) throw std::invalid_argument("WorkerPool: workers must be >= 1");
  Grid2D out(phi.nx, phi.ny, phi.dx, phi.dy);
  detail::check(sg_weno_advect(phi.data(), vel.u.data(), vel.v.data(), phi.nx, phi.ny, phi.dx, phi.dy, out.data(),
                               SG_MEM_HOST, nullptr));
  return out;
}

}  // namespace stengrid
