// The closed-form tail of graspmatch::icp_closed_form_step (optim.cpp:64-90):
// 3x3 one-sided Jacobi SVD exactly as the reference is built (the
// oracle/shim/Eigen/Dense JacobiSVD: sweeps over (p, q) column pairs,
// descending stable order, orthonormal completion of vanishing columns), the
// Kabsch reflection guard and Shepperd's quaternion extraction
// (optim.cpp:29-46).  FP64 in the reference's operation order (-fmad=false).
#pragma once

#include "dmath.cuh"

namespace asicp {

struct Mat3 {
  double a[3][3];  // a[row][col]
};

// Shim matrix product: (i, j) = a(i,0) b(0,j) + a(i,1) b(1,j) + a(i,2) b(2,j), left to right.
ASICP_HD Mat3 mm3(const Mat3& x, const Mat3& y) {
  Mat3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.a[i][j] = (x.a[i][0] * y.a[0][j] + x.a[i][1] * y.a[1][j]) + x.a[i][2] * y.a[2][j];
  return o;
}
ASICP_HD Mat3 tr3(const Mat3& x) {
  Mat3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.a[i][j] = x.a[j][i];
  return o;
}
// Shim determinant (3x3 cofactor expansion down the first column).
ASICP_HD double det3(const Mat3& m) {
  const auto c = [&](int i, int j) { return m.a[i][j]; };
  return (c(0, 0) * (c(1, 1) * c(2, 2) - c(1, 2) * c(2, 1)) - c(1, 0) * (c(0, 1) * c(2, 2) - c(0, 2) * c(2, 1))) +
         c(2, 0) * (c(0, 1) * c(1, 2) - c(0, 2) * c(1, 1));
}

// Eigen::JacobiSVD<Mat3>(a, ComputeFullU | ComputeFullV) as the shim computes it.
ASICP_HD void svd3(const Mat3& in, double sing[3], Mat3& U, Mat3& V) {
  Mat3 u = in, v = {{{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}}};
  for (int sweep = 0; sweep < 100; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int k = 0; k < 3; ++k) {
          alpha += u.a[k][p] * u.a[k][p];
          beta += u.a[k][q] * u.a[k][q];
          gamma += u.a[k][p] * u.a[k][q];
        }
        if (fabs(gamma) <= 1e-300 || fabs(gamma) <= 1e-17 * sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int k = 0; k < 3; ++k) {
          const double up = u.a[k][p], uq = u.a[k][q];
          u.a[k][p] = c * up - s * uq;
          u.a[k][q] = s * up + c * uq;
          const double vp = v.a[k][p], vq = v.a[k][q];
          v.a[k][p] = c * vp - s * vq;
          v.a[k][q] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  double sv[3];
  for (int j = 0; j < 3; ++j) {
    double s2 = 0.0;
    for (int k = 0; k < 3; ++k) s2 += u.a[k][j] * u.a[k][j];
    sv[j] = sqrt(s2);
  }
  // std::sort of 3 indices by descending sv: libstdc++ insertion sort (stable).
  int order[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i) {
    const int val = order[i];
    int j = i;
    while (j > 0 && sv[val] > sv[order[j - 1]]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = val;
  }
  const double tiny = 1e-300;
  for (int i = 0; i < 3; ++i) {
    const int j = order[i];
    sing[i] = sv[j];
    for (int k = 0; k < 3; ++k) {
      V.a[k][i] = v.a[k][j];
      U.a[k][i] = sv[j] > tiny ? u.a[k][j] / sv[j] : 0.0;
    }
  }
  for (int i = 0; i < 3; ++i) {
    if (sing[i] > tiny * (1.0 < sing[0] ? sing[0] : 1.0) && sing[i] > 0.0) continue;  // std::max(1.0, s0)
    for (int trial = 0; trial < 3; ++trial) {
      double cand[3] = {trial == 0 ? 1.0 : 0.0, trial == 1 ? 1.0 : 0.0, trial == 2 ? 1.0 : 0.0};
      for (int k = 0; k < 3; ++k) {
        if (k == i) continue;
        if (k > i && !(sing[k] > 0.0)) continue;
        const double proj = (U.a[0][k] * cand[0] + U.a[1][k] * cand[1]) + U.a[2][k] * cand[2];
        for (int r = 0; r < 3; ++r) cand[r] = cand[r] - U.a[r][k] * proj;
      }
      const double n = sqrt((cand[0] * cand[0] + cand[1] * cand[1]) + cand[2] * cand[2]);
      if (n > 1e-6) {
        for (int r = 0; r < 3; ++r) U.a[r][i] = cand[r] / n;
        break;
      }
    }
  }
}

// optim.cpp:29-46 quaternion_from_matrix (Shepperd), then normalized_quaternion.
ASICP_HD Q4 quaternion_from_matrix(const Mat3& m) {
  const auto r = [&](int i, int j) { return m.a[i][j]; };
  const double tr = (r(0, 0) + r(1, 1)) + r(2, 2);
  Q4 q;
  if (tr > 0.0) {
    const double s = sqrt(tr + 1.0) * 2.0;
    q = Q4{0.25 * s, (r(2, 1) - r(1, 2)) / s, (r(0, 2) - r(2, 0)) / s, (r(1, 0) - r(0, 1)) / s};
  } else if (r(0, 0) > r(1, 1) && r(0, 0) > r(2, 2)) {
    const double s = sqrt(((1.0 + r(0, 0)) - r(1, 1)) - r(2, 2)) * 2.0;
    q = Q4{(r(2, 1) - r(1, 2)) / s, 0.25 * s, (r(0, 1) + r(1, 0)) / s, (r(0, 2) + r(2, 0)) / s};
  } else if (r(1, 1) > r(2, 2)) {
    const double s = sqrt(((1.0 + r(1, 1)) - r(0, 0)) - r(2, 2)) * 2.0;
    q = Q4{(r(0, 2) - r(2, 0)) / s, (r(0, 1) + r(1, 0)) / s, 0.25 * s, (r(1, 2) + r(2, 1)) / s};
  } else {
    const double s = sqrt(((1.0 + r(2, 2)) - r(0, 0)) - r(1, 1)) * 2.0;
    q = Q4{(r(1, 0) - r(0, 1)) / s, (r(0, 2) + r(2, 0)) / s, (r(1, 2) + r(2, 1)) / s, 0.25 * s};
  }
  return normalized(q);
}

// optim.cpp:64-89 from the means and the covariance: theta_out (t, q) and the
// degenerate flag.  th = the input pose (t, q).
ASICP_HD int kabsch_finish(const double* th, V3 src_mean, V3 ref_mean, const Mat3& cov, long long n, double* out) {
  double sing[3];
  Mat3 U, V;
  svd3(cov, sing, U, V);
  if (n < 3 || sing[1] <= 1e-12 * (1.0 < sing[0] ? sing[0] : 1.0)) {
    const M3 R = rotation_matrix(pose_q(th));
    const V3 moved = add(mul(R, src_mean), pose_t(th));
    const V3 d = sub(ref_mean, moved);
    out[0] = th[0] + d.x;
    out[1] = th[1] + d.y;
    out[2] = th[2] + d.z;
    for (int i = 3; i < 7; ++i) out[i] = th[i];
    return 1;
  }
  const Mat3 Ut = tr3(U);
  Mat3 D = {{{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}}};
  D.a[2][2] = det3(mm3(V, Ut)) < 0.0 ? -1.0 : 1.0;
  const Mat3 r = mm3(mm3(V, D), Ut);
  const Q4 q = quaternion_from_matrix(r);
  M3 rm;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) rm.m[3 * i + j] = r.a[i][j];
  const V3 t = sub(ref_mean, mul(rm, src_mean));
  out[0] = t.x;
  out[1] = t.y;
  out[2] = t.z;
  out[3] = q.w;
  out[4] = q.x;
  out[5] = q.y;
  out[6] = q.z;
  return 0;
}

}  // namespace asicp
