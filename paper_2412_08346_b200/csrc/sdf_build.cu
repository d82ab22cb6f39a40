// graspmatch::build_sdf (sdf.cpp:48-175) on the B200 — SURVEY.md §8(f) rank 1.
//
//   * node distances: exact FP64 brute force, dist = float(sqrt(min_p
//     (p - node).squaredNorm())) (the kd-tree's answer, spatial_index.cpp:
//     61-71, 100-104; ties do not matter for a distance), the cloud staged in
//     shared memory tile by tile, one node per thread;
//   * sign: the widest-path (max-min) clearance from the grid boundary
//     (sdf.cpp:96-142) is the unique fixpoint of
//       c[v] = max(c[v], min(dist[v], max_{u ~ v} c[u])),  c[boundary] = dist,
//     reached by in-place relaxation sweeps (values only grow, so any order
//     converges to the same floats as the reference's priority queue);
//   * values and the boundary maximum exactly as sdf.cpp:150-173.
// Validation and the grid geometry (bounds, dims, sample spacing, skin) are
// host work, identical to the reference's.
#include "asicp.h"
#include "common.cuh"
#include "kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace asicp {
namespace {

constexpr int kSdfThreads = 256;
constexpr int kSdfTile = 1024;

__global__ void __launch_bounds__(kSdfThreads) sdf_dist_kernel(const double* cloud, int n, double ox, double oy,
                                                               double oz, double voxel, int nx, int ny, int nz,
                                                               float* dist) {
  __shared__ double px[kSdfTile], py[kSdfTile], pz[kSdfTile];
  const int64_t total = static_cast<int64_t>(nx) * ny * nz;
  const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool valid = id < total;
  const int iz = valid ? static_cast<int>(id % nz) : 0;
  const int iy = valid ? static_cast<int>((id / nz) % ny) : 0;
  const int ix = valid ? static_cast<int>(id / (static_cast<int64_t>(ny) * nz)) : 0;
  // node_position (sdf.hpp:33-35): origin + voxel * (ix, iy, iz)
  const V3 q = V3{ox + voxel * static_cast<double>(ix), oy + voxel * static_cast<double>(iy),
                  oz + voxel * static_cast<double>(iz)};
  double best = INFINITY;
  for (int t0 = 0; t0 < n; t0 += kSdfTile) {
    const int nt = min(kSdfTile, n - t0);
    __syncthreads();
    for (int k = threadIdx.x; k < nt; k += blockDim.x) {
      px[k] = cloud[3 * static_cast<int64_t>(t0 + k)];
      py[k] = cloud[3 * static_cast<int64_t>(t0 + k) + 1];
      pz[k] = cloud[3 * static_cast<int64_t>(t0 + k) + 2];
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < nt; ++k) {
      const double d2 = sqnorm(sub(V3{px[k], py[k], pz[k]}, q));  // (points[idx] - query).squaredNorm()
      best = d2 < best ? d2 : best;
    }
  }
  if (valid) dist[id] = static_cast<float>(sqrt(best));
}

__device__ __forceinline__ bool on_boundary(int ix, int iy, int iz, int nx, int ny, int nz) {
  return ix == 0 || iy == 0 || iz == 0 || ix == nx - 1 || iy == ny - 1 || iz == nz - 1;
}

__global__ void sdf_clear_init_kernel(const float* dist, float* clr, int nx, int ny, int nz) {
  const int64_t total = static_cast<int64_t>(nx) * ny * nz;
  for (int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; id < total;
       id += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int iz = static_cast<int>(id % nz), iy = static_cast<int>((id / nz) % ny),
              ix = static_cast<int>(id / (static_cast<int64_t>(ny) * nz));
    clr[id] = on_boundary(ix, iy, iz, nx, ny, nz) ? fmaxf(dist[id], 0.0f) : 0.0f;
  }
}

// One in-place relaxation sweep; *changed is set when any node grew.
__global__ void sdf_relax_kernel(const float* dist, float* clr, int nx, int ny, int nz, int* changed) {
  const int64_t total = static_cast<int64_t>(nx) * ny * nz;
  bool any = false;
  for (int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; id < total;
       id += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int iz = static_cast<int>(id % nz), iy = static_cast<int>((id / nz) % ny),
              ix = static_cast<int>(id / (static_cast<int64_t>(ny) * nz));
    if (on_boundary(ix, iy, iz, nx, ny, nz)) continue;  // already at their maximum, dist
    const int64_t sx = static_cast<int64_t>(ny) * nz, sy = nz;
    volatile const float* c = clr;
    float m = fmaxf(fmaxf(fmaxf(c[id - sx], c[id + sx]), fmaxf(c[id - sy], c[id + sy])), fmaxf(c[id - 1], c[id + 1]));
    const float cand = fminf(m, dist[id]);
    if (cand > clr[id]) {
      clr[id] = cand;
      any = true;
    }
  }
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *changed = 1;
}

__global__ void sdf_values_kernel(const float* dist, const float* clr, float skin, int nx, int ny, int nz,
                                  float* values, unsigned int* boundary_max_bits) {
  const int64_t total = static_cast<int64_t>(nx) * ny * nz;
  for (int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; id < total;
       id += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    constexpr float kEscapeRatio = 0.9f;  // sdf.cpp:150
    const bool exterior = clr[id] >= kEscapeRatio * dist[id];
    const float v = exterior ? -dist[id] : dist[id] - skin;
    values[id] = v;
    const int iz = static_cast<int>(id % nz), iy = static_cast<int>((id / nz) % ny),
              ix = static_cast<int>(id / (static_cast<int64_t>(ny) * nz));
    if (on_boundary(ix, iy, iz, nx, ny, nz)) atomicMax(boundary_max_bits, __float_as_uint(fabsf(v)));
  }
}

struct SdfArgError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Smallest / largest eigenvalue of a symmetric 3x3 matrix by cyclic Jacobi
// rotations (an exactly decoupled zero direction stays exactly zero, as in
// the reference's SelfAdjointEigenSolver).
void sym3_eig_extremes(const double a_in[3][3], double* lo, double* hi) {
  double a[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = a_in[i][j];
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    const double diag = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
    if (off == 0.0 || off <= 1e-36 * diag) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- A J (columns p, q)
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {  // A <- J^T A (rows p, q)
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        a[p][q] = a[q][p] = 0.0;
      }
  }
  *lo = std::min({a[0][0], a[1][1], a[2][2]});
  *hi = std::max({a[0][0], a[1][1], a[2][2]});
}

// sdf.cpp:37-44
bool coplanar(const double* cloud, int64_t n) {
  if (n < 4) return true;
  double c[3] = {0.0, 0.0, 0.0};
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) c[a] = c[a] + cloud[3 * i + a];
  for (int a = 0; a < 3; ++a) c[a] = c[a] / static_cast<double>(n);
  double cov[3][3] = {};
  for (int64_t i = 0; i < n; ++i) {
    const double d[3] = {cloud[3 * i] - c[0], cloud[3 * i + 1] - c[1], cloud[3 * i + 2] - c[2]};
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) cov[r][s] += d[r] * d[s];
  }
  double lo = 0.0, hi = 0.0;
  sym3_eig_extremes(cov, &lo, &hi);
  return lo <= 1e-18 * std::max(1.0, hi);
}

// sdf.cpp:21-35
double sample_spacing(const double* cloud, int64_t n) {
  std::vector<double> nn;
  const int64_t stride = std::max<int64_t>(1, n / 512);
  for (int64_t i = 0; i < n; i += stride) {
    double best = std::numeric_limits<double>::infinity();
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const double dx = cloud[3 * i] - cloud[3 * j], dy = cloud[3 * i + 1] - cloud[3 * j + 1],
                   dz = cloud[3 * i + 2] - cloud[3 * j + 2];
      best = std::min(best, (dx * dx + dy * dy) + dz * dz);
    }
    nn.push_back(std::sqrt(best));
  }
  std::sort(nn.begin(), nn.end());
  return nn.empty() ? 0.0 : nn[static_cast<size_t>(0.95 * static_cast<double>(nn.size() - 1))];
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("asicp_build_sdf: ") + what + ": " + cudaGetErrorString(e));
}

}  // namespace

int build_sdf_device(int device, cudaStream_t st, const double* cloud, int64_t n, double voxel, double padding_opt,
                     double band, int32_t* dims, double* meta, float* values, std::string* err) {
  if (!(voxel > 0.0)) {
    *err = "build_sdf: voxel must be positive";
    return ASICP_INVALID_ARGUMENT;
  }
  if (n < 4 || coplanar(cloud, n)) {
    *err = "build_sdf: need >= 4 non-coplanar points";
    return ASICP_INVALID_ARGUMENT;
  }
  const double padding = padding_opt >= 0.0 ? padding_opt : 4.0 * voxel;
  double lo[3] = {cloud[0], cloud[1], cloud[2]}, hi[3] = {cloud[0], cloud[1], cloud[2]};
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], cloud[3 * i + a]);
      hi[a] = std::max(hi[a], cloud[3 * i + a]);
    }
  for (int a = 0; a < 3; ++a) {
    lo[a] = lo[a] - padding;
    hi[a] = hi[a] + padding;
    dims[a] = static_cast<int32_t>(std::ceil((hi[a] - lo[a]) / voxel)) + 1;
    meta[a] = lo[a];
  }
  meta[3] = voxel;
  meta[4] = 0.0;
  if (!values) return ASICP_OK;
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  const int64_t total = static_cast<int64_t>(nx) * ny * nz;
  const double spacing = sample_spacing(cloud, n);
  const double closure = 1.05 * std::sqrt(0.25 * voxel * voxel + 0.5 * spacing * spacing);
  const double skin = std::max(band, closure);

  check(cudaSetDevice(device), "cudaSetDevice");
  double* d_cloud = nullptr;
  float *d_dist = nullptr, *d_clr = nullptr, *d_val = nullptr;
  int* d_changed = nullptr;
  unsigned int* d_bmax = nullptr;
  auto release = [&] {
    cudaFree(d_cloud);
    cudaFree(d_dist);
    cudaFree(d_clr);
    cudaFree(d_val);
    cudaFree(d_changed);
    cudaFree(d_bmax);
  };
  try {
    check(cudaMalloc(&d_cloud, static_cast<size_t>(n) * 24), "cudaMalloc");
    check(cudaMalloc(&d_dist, static_cast<size_t>(total) * 4), "cudaMalloc");
    check(cudaMalloc(&d_clr, static_cast<size_t>(total) * 4), "cudaMalloc");
    check(cudaMalloc(&d_val, static_cast<size_t>(total) * 4), "cudaMalloc");
    check(cudaMalloc(&d_changed, 4), "cudaMalloc");
    check(cudaMalloc(&d_bmax, 4), "cudaMalloc");
    check(cudaMemcpyAsync(d_cloud, cloud, static_cast<size_t>(n) * 24, cudaMemcpyHostToDevice, st), "H2D");
    const int blocks = static_cast<int>((total + kSdfThreads - 1) / kSdfThreads);
    sdf_dist_kernel<<<blocks, kSdfThreads, 0, st>>>(d_cloud, static_cast<int>(n), lo[0], lo[1], lo[2], voxel, nx, ny,
                                                    nz, d_dist);
    sdf_clear_init_kernel<<<592, 256, 0, st>>>(d_dist, d_clr, nx, ny, nz);
    // Relaxation until a batch of sweeps changes nothing.
    for (int round = 0;; ++round) {
      check(cudaMemsetAsync(d_changed, 0, 4, st), "memset");
      for (int s = 0; s < 8; ++s) sdf_relax_kernel<<<592, 256, 0, st>>>(d_dist, d_clr, nx, ny, nz, d_changed);
      int changed = 0;
      check(cudaMemcpyAsync(&changed, d_changed, 4, cudaMemcpyDeviceToHost, st), "D2H");
      check(cudaStreamSynchronize(st), "sync");
      if (!changed) break;
      if (round > 1000000) throw std::runtime_error("asicp_build_sdf: clearance relaxation did not converge");
    }
    check(cudaMemsetAsync(d_bmax, 0, 4, st), "memset");
    sdf_values_kernel<<<592, 256, 0, st>>>(d_dist, d_clr, static_cast<float>(skin), nx, ny, nz, d_val, d_bmax);
    unsigned int bmax_bits = 0;
    check(cudaMemcpyAsync(values, d_val, static_cast<size_t>(total) * 4, cudaMemcpyDeviceToHost, st), "D2H");
    check(cudaMemcpyAsync(&bmax_bits, d_bmax, 4, cudaMemcpyDeviceToHost, st), "D2H");
    check(cudaStreamSynchronize(st), "sync");
    float bmax;
    std::memcpy(&bmax, &bmax_bits, 4);
    meta[4] = static_cast<double>(bmax);
  } catch (...) {
    release();
    throw;
  }
  release();
  return ASICP_OK;
}

}  // namespace asicp
