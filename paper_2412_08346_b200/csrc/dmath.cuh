// FP64 pose / geometry algebra in the reference's exact operation order.
//
// Every function mirrors one reference function and evaluates its
// arithmetic in the same order as the reference compiled against
// oracle/shim/Eigen (left-to-right reductions, no fused multiply-add: this
// translation unit is compiled with -fmad=false, and the reference oracle
// with no -march, so neither side contracts a*b+c).  That is what makes the
// device trajectory bit-identical to graspmatch::optimize_grasp.
#pragma once

#include <cmath>
#include <cstdint>

#define ASICP_HD __host__ __device__ __forceinline__

namespace asicp {

struct V3 {
  double x, y, z;
};
struct Q4 {
  double w, x, y, z;
};
struct M3 {
  double m[9];  // row-major
  ASICP_HD double operator()(int r, int c) const { return m[3 * r + c]; }
};

ASICP_HD V3 v3(double x, double y, double z) { return V3{x, y, z}; }
ASICP_HD V3 add(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
ASICP_HD V3 sub(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
ASICP_HD V3 neg(V3 a) { return V3{-a.x, -a.y, -a.z}; }
// squaredNorm: ((x*x + y*y) + z*z)
ASICP_HD double sqnorm(V3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
ASICP_HD double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
ASICP_HD double sqnorm4(Q4 q) { return ((q.w * q.w + q.x * q.x) + q.y * q.y) + q.z * q.z; }

// Matrix * vector, each coefficient a left-to-right dot of the row.
ASICP_HD V3 mul(const M3& r, V3 p) {
  return V3{(r.m[0] * p.x + r.m[1] * p.y) + r.m[2] * p.z, (r.m[3] * p.x + r.m[4] * p.y) + r.m[5] * p.z,
            (r.m[6] * p.x + r.m[7] * p.y) + r.m[8] * p.z};
}

// geometry.cpp:8-15 rotation_matrix_homogeneous
ASICP_HD M3 rotation_matrix_homogeneous(Q4 q) {
  const double w = q.w, x = q.x, y = q.y, z = q.z;
  M3 r;
  r.m[0] = w * w + x * x - y * y - z * z;
  r.m[1] = 2.0 * (x * y - w * z);
  r.m[2] = 2.0 * (x * z + w * y);
  r.m[3] = 2.0 * (x * y + w * z);
  r.m[4] = w * w - x * x + y * y - z * z;
  r.m[5] = 2.0 * (y * z - w * x);
  r.m[6] = 2.0 * (x * z - w * y);
  r.m[7] = 2.0 * (y * z + w * x);
  r.m[8] = w * w - x * x - y * y + z * z;
  return r;
}

// geometry.cpp:17-21 rotation_matrix (unit check is done on the host for the
// initial poses; every device update renormalises, optim.cpp:112, 233).
ASICP_HD M3 rotation_matrix(Q4 q) {
  const double n2 = sqnorm4(q);
  M3 r = rotation_matrix_homogeneous(q);
  for (int i = 0; i < 9; ++i) r.m[i] = r.m[i] / n2;
  return r;
}

// geometry.cpp:23-32 rotation_matrix_derivatives: d[j] = 2 * (row-major comma list).
ASICP_HD void rotation_matrix_derivatives(Q4 q, M3 d[4]) {
  const double w = q.w, x = q.x, y = q.y, z = q.z;
  const double a0[9] = {w, -z, y, z, w, -x, -y, x, w};
  const double a1[9] = {x, y, z, y, -x, -w, z, w, -x};
  const double a2[9] = {-y, x, w, x, y, z, -w, z, -y};
  const double a3[9] = {-z, -w, x, w, -z, y, x, y, z};
  for (int i = 0; i < 9; ++i) {
    d[0].m[i] = a0[i] * 2.0;
    d[1].m[i] = a1[i] * 2.0;
    d[2].m[i] = a2[i] * 2.0;
    d[3].m[i] = a3[i] * 2.0;
  }
}

// geometry.cpp:68-74: R p + t
ASICP_HD V3 transform(const M3& r, V3 t, V3 p) { return add(mul(r, p), t); }

// geometry.cpp:80-85 inverse: q^-1 = (w,-x,-y,-z), t^-1 = -(R(q^-1) t)
ASICP_HD void inverse(Q4 q, V3 t, Q4* qi, V3* ti) {
  *qi = Q4{q.w, -q.x, -q.y, -q.z};
  *ti = neg(mul(rotation_matrix(*qi), t));
}

// geometry.cpp:234 normalized_quaternion: q / ||q||
ASICP_HD Q4 normalized(Q4 q) {
  const double n = sqrt(sqnorm4(q));
  return Q4{q.w / n, q.x / n, q.y / n, q.z / n};
}

// std::clamp(v, lo, hi)
ASICP_HD double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// SDF grid view (sdf.hpp:23-39).
struct Grid {
  int32_t dims[3];
  double origin[3];
  double voxel;
  double boundary_max_abs;
  double offset[3];
  int64_t values_offset;  // into the concatenated value buffer
  double lip;             // max |node difference| / voxel along any axis (FP32 pre-test bound)
  double vmax;            // max |value|
  int32_t cdims[3];       // coarse blocks of 4x4x4 cells per axis
  int64_t coarse_offset;  // into the concatenated coarse-max buffer
};

constexpr int kCoarse = 4;  // cells per coarse block edge

// sdf.cpp:177-203 query(SdfGrid, p) in the reference order.
ASICP_HD double sdf_query(const Grid& g, const float* values, double px, double py, double pz) {
  const double p[3] = {px, py, pz};
  double hi[3];
  for (int a = 0; a < 3; ++a) hi[a] = g.origin[a] + g.voxel * static_cast<double>(g.dims[a] - 1);
  const bool outside = (p[0] < g.origin[0] || p[1] < g.origin[1] || p[2] < g.origin[2]) ||
                       (p[0] > hi[0] || p[1] > hi[1] || p[2] > hi[2]);
  if (outside) {
    double d[3];
    for (int a = 0; a < 3; ++a) {
      // p.cwiseMax(origin).cwiseMin(hi) with std::max/std::min semantics.
      double c = p[a] < g.origin[a] ? g.origin[a] : p[a];
      c = hi[a] < c ? hi[a] : c;
      d[a] = p[a] - c;
    }
    const double n = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    return -(n + g.boundary_max_abs);
  }
  double local[3];
  for (int a = 0; a < 3; ++a) local[a] = (p[a] - g.origin[a]) / g.voxel;
  int ix = static_cast<int>(local[0]);
  int iy = static_cast<int>(local[1]);
  int iz = static_cast<int>(local[2]);
  ix = ix < g.dims[0] - 2 ? ix : g.dims[0] - 2;
  iy = iy < g.dims[1] - 2 ? iy : g.dims[1] - 2;
  iz = iz < g.dims[2] - 2 ? iz : g.dims[2] - 2;
  ix = ix > 0 ? ix : 0;
  iy = iy > 0 ? iy : 0;
  iz = iz > 0 ? iz : 0;
  const double fx = clampd(local[0] - ix, 0.0, 1.0);
  const double fy = clampd(local[1] - iy, 0.0, 1.0);
  const double fz = clampd(local[2] - iz, 0.0, 1.0);
  const int ny = g.dims[1], nz = g.dims[2];
  auto v = [&](int dx, int dy, int dz) {
    const int64_t id = (static_cast<int64_t>(ix + dx) * ny + (iy + dy)) * nz + (iz + dz);
    return static_cast<double>(values[g.values_offset + id]);
  };
  const double c00 = v(0, 0, 0) * (1 - fx) + v(1, 0, 0) * fx;
  const double c01 = v(0, 0, 1) * (1 - fx) + v(1, 0, 1) * fx;
  const double c10 = v(0, 1, 0) * (1 - fx) + v(1, 1, 0) * fx;
  const double c11 = v(0, 1, 1) * (1 - fx) + v(1, 1, 1) * fx;
  const double c0 = c00 * (1 - fy) + c10 * fy;
  const double c1 = c01 * (1 - fy) + c11 * fy;
  return c0 * (1 - fz) + c1 * fz;
}

// Particle pose helpers: theta = (tx, ty, tz, qw, qx, qy, qz).
ASICP_HD V3 pose_t(const double* th) { return V3{th[0], th[1], th[2]}; }
ASICP_HD Q4 pose_q(const double* th) { return Q4{th[3], th[4], th[5], th[6]}; }

}  // namespace asicp
