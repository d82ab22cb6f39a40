// Collision test of optimize_grasp on the B200: colliding_points
// (sdf.cpp:227-243) with query(stacked) (sdf.cpp:220-225) and the trilinear
// query (sdf.cpp:177-203) — for every particle, the scene points whose SDF
// value in the particle's gripper frame exceeds contact_tolerance, in scene
// order (grasp.cpp:176-181).
//
// Scene layout (built on the device once per asicp_prepare):
//   * scene32: the points rounded to FP32, w = |p|_1 rounded up (the pre-test
//     transform-error margin), original order;
//   * the points sorted along a 30-bit Morton curve (cub radix sort, stable:
//     deterministic) and cut into clusters of 32 consecutive points, each cut
//     into 4 sub-clusters of 8; per (sub-)cluster an FP32 centre c and a
//     radius r >= max |p - c| (FP64, rounded up), plus the sorted copy of the
//     FP32 points and the permutation back to scene order.
//
// Per particle (one CTA):
//   1. cluster test, one thread per cluster, then the same test on the
//      sub-clusters of the clusters it does not clear: the centre is transformed in FP32
//      (error <= delta per axis).  Every point of the cluster lies within
//      r + delta of the transformed centre, so the cluster is clear when
//        - it lies outside the grid box by more than r + delta along an axis
//          (then every point is outside, where the reference returns
//          -(distance + boundary_max_abs) <= contact_tolerance), or
//        - with c' the centre clamped to the box, the FP32 trilinear value at
//          c' plus its rounding margin plus lip * (sqrt(3) r + 3 delta) is at
//          most the tolerance: inside the box the interpolant is Lipschitz
//          with per-axis slope <= lip (the largest node difference / voxel),
//          clamping to the box does not increase the L1 distance to a point
//          inside it, and points outside the box cannot collide (above);
//   2. points of the remaining clusters, one lane per point: the per-point
//      FP32 pre-test with rigorous margins (outside the box -> clear; inside
//      -> a dilated 4^3-block maximum, then the FP32 trilinear value +- a
//      Lipschitz margin), the exact FP64 reference evaluation for the few
//      points the pre-test cannot decide; hits set a bit of a shared bitmask
//      indexed by the ORIGINAL scene position;
//   3. the bitmask is compacted in scene order (warp ballots / popcounts).
// When contact_tolerance < -boundary_max_abs points outside the box can
// collide: the cluster test is skipped and every point takes step 2.
#include "common.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace asicp {

// ---------------------------------------------------------------------------
// Scene preparation (asicp_prepare).
// ---------------------------------------------------------------------------
__global__ void scene32_kernel(const double* scene64, int n, float4* s32) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float x = __double2float_rn(scene64[3 * i]), y = __double2float_rn(scene64[3 * i + 1]),
              z = __double2float_rn(scene64[3 * i + 2]);
  const double l1 = (fabs(static_cast<double>(x)) + fabs(static_cast<double>(y))) + fabs(static_cast<double>(z));
  s32[i] = make_float4(x, y, z, nextafterf(__double2float_rn(l1), INFINITY));
}

// Bounding box of the scene (one CTA): box[0..2] = min, box[3..5] = max.
__global__ void __launch_bounds__(1024) scene_box_kernel(const double* scene64, int n, double* box) {
  __shared__ double red[6][32];
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int a = 0; a < 3; ++a) {
      const double v = scene64[3 * i + a];
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
  for (int o = 16; o > 0; o >>= 1)
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int a = 0; a < 3; ++a) {
      red[a][w] = lo[a];
      red[3 + a][w] = hi[a];
    }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int a = threadIdx.x;
    double v = red[a][0];
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) v = a < 3 ? fmin(v, red[a][k]) : fmax(v, red[a][k]);
    box[a] = v;
  }
}

__device__ __forceinline__ unsigned int spread10(unsigned int v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void scene_morton_kernel(const double* scene64, int n, const double* box, unsigned int* code, int* idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned int q[3];
  for (int a = 0; a < 3; ++a) {
    const double ext = box[3 + a] - box[a];
    const double s = ext > 0.0 ? 1023.0 / ext : 0.0;
    const double u = (scene64[3 * i + a] - box[a]) * s;
    q[a] = static_cast<unsigned int>(fmin(fmax(u, 0.0), 1023.0));
  }
  code[i] = spread10(q[0]) | (spread10(q[1]) << 1) | (spread10(q[2]) << 2);
  idx[i] = i;
}

// Centre (FP32 of the FP64 box midpoint) and radius >= max |p - c| (FP64,
// rounded up) of sorted points [i0, i1); an empty range gets radius 0.
__device__ float4 bound_sphere(const double* scene64, const int* perm, int i0, int i1) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = i0; i < i1; ++i) {
    const int o = perm[i];
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], scene64[3 * o + a]);
      hi[a] = fmax(hi[a], scene64[3 * o + a]);
    }
  }
  if (i1 <= i0) return make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  float cf[3];
  for (int a = 0; a < 3; ++a) cf[a] = __double2float_rn(0.5 * (lo[a] + hi[a]));
  double r2 = 0.0;
  for (int i = i0; i < i1; ++i) {
    const int o = perm[i];
    const double dx = scene64[3 * o] - cf[0], dy = scene64[3 * o + 1] - cf[1], dz = scene64[3 * o + 2] - cf[2];
    r2 = fmax(r2, dx * dx + dy * dy + dz * dz);
  }
  // sqrt and the float conversion rounded up, plus slack for the FP64 sums.
  const float r = __double2float_ru(__dsqrt_ru(r2) * (1.0 + 1e-12)) * (1.0f + 1e-6f) + 1e-12f;
  return make_float4(cf[0], cf[1], cf[2], r);
}

// One thread per cluster of kClusterPts sorted points: its bounding sphere and
// those of its kSubPerCluster sub-clusters of kSubPts, the sorted FP32 points
// and the permutation (-1 pads the last cluster).
__global__ void scene_cluster_kernel(const double* scene64, const float4* s32, const int* perm, int n,
                                     float4* clusters, float4* subclusters, float4* s32s, int* perm_pad,
                                     int n_clusters) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_clusters) return;
  const int i0 = c * kClusterPts, i1 = min(n, i0 + kClusterPts);
  clusters[c] = bound_sphere(scene64, perm, i0, i1);
  for (int k = 0; k < kSubPerCluster; ++k) {
    const int a = min(i1, i0 + k * kSubPts), b = min(i1, a + kSubPts);
    subclusters[c * kSubPerCluster + k] = bound_sphere(scene64, perm, a, b);
  }
  for (int k = 0; k < kClusterPts; ++k) {
    const int i = i0 + k;
    if (i < i1) {
      s32s[i] = s32[perm[i]];
      perm_pad[i] = perm[i];
    } else {
      s32s[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      perm_pad[i] = -1;
    }
  }
}

size_t scene_sort_temp_bytes(int n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const unsigned int*>(nullptr),
                                  static_cast<unsigned int*>(nullptr), static_cast<const int*>(nullptr),
                                  static_cast<int*>(nullptr), n, 0, 30);
  return bytes;
}

void launch_scene_prepare(const double* scene64, int n, float4* s32, double* box, unsigned int* code_in,
                          unsigned int* code_out, int* idx_in, int* perm, void* temp, size_t temp_bytes,
                          float4* clusters, float4* subclusters, float4* s32s, int* perm_pad, cudaStream_t st) {
  const int nb = ceil_div(n, 256);
  scene32_kernel<<<nb, 256, 0, st>>>(scene64, n, s32);
  scene_box_kernel<<<1, 1024, 0, st>>>(scene64, n, box);
  scene_morton_kernel<<<nb, 256, 0, st>>>(scene64, n, box, code_in, idx_in);
  size_t bytes = temp_bytes;
  if (cub::DeviceRadixSort::SortPairs(temp, bytes, code_in, code_out, idx_in, perm, n, 0, 30, st) != cudaSuccess)
    throw std::runtime_error("asicp: scene sort failed");
  const int ncl = ceil_div(n, kClusterPts);
  scene_cluster_kernel<<<ceil_div(ncl, 128), 128, 0, st>>>(scene64, s32, perm, n, clusters, subclusters, s32s,
                                                            perm_pad, ncl);
}

// ---------------------------------------------------------------------------
// The collision kernel.
// ---------------------------------------------------------------------------
constexpr int kColThreads = 128;
constexpr int kColWarps = kColThreads / 32;
constexpr int kColU = 2;  // warp steps batched in the point test

// The exact FP64 test of one scene point (colliding_points body,
// sdf.cpp:237-239), kept out of line so its register needs do not throttle
// the FP32 pre-test.
__device__ __noinline__ bool collide_exact(const double* th, const Grid* gp, const float* values, const double* p64,
                                           double tol) {
  const Grid& g = *gp;
  Q4 qi;
  V3 ti;
  inverse(pose_q(th), pose_t(th), &qi, &ti);
  const M3 r = rotation_matrix(qi);
  const V3 off = V3{g.offset[0], g.offset[1], g.offset[2]};
  const V3 local = sub(add(add(mul(r, V3{p64[0], p64[1], p64[2]}), ti), off), off);
  return sdf_query(g, values, local.x, local.y, local.z) > tol;
}

__device__ __forceinline__ float tri32(const Grid& g, const float* vals, float ux, float uy, float uz) {
  const int ix = max(min(static_cast<int>(ux), g.dims[0] - 2), 0);
  const int iy = max(min(static_cast<int>(uy), g.dims[1] - 2), 0);
  const int iz = max(min(static_cast<int>(uz), g.dims[2] - 2), 0);
  const float fxx = fminf(fmaxf(ux - ix, 0.0f), 1.0f), fyy = fminf(fmaxf(uy - iy, 0.0f), 1.0f),
              fzz = fminf(fmaxf(uz - iz, 0.0f), 1.0f);
  const float* v0 = vals + (static_cast<int64_t>(ix) * g.dims[1] + iy) * g.dims[2] + iz;
  const int sy = g.dims[2], sx = g.dims[1] * g.dims[2];
  const float c00 = __fmaf_rn(fxx, __ldg(v0 + sx) - __ldg(v0), __ldg(v0));
  const float c01 = __fmaf_rn(fxx, __ldg(v0 + sx + 1) - __ldg(v0 + 1), __ldg(v0 + 1));
  const float c10 = __fmaf_rn(fxx, __ldg(v0 + sx + sy) - __ldg(v0 + sy), __ldg(v0 + sy));
  const float c11 = __fmaf_rn(fxx, __ldg(v0 + sx + sy + 1) - __ldg(v0 + sy + 1), __ldg(v0 + sy + 1));
  const float c0 = __fmaf_rn(fyy, c10 - c00, c00);
  const float c1 = __fmaf_rn(fyy, c11 - c01, c01);
  return __fmaf_rn(fzz, c1 - c0, c0);
}

// Cluster test (comment at the top of the file): true when no point within
// cl.w of the centre cl.xyz can collide.
__device__ __forceinline__ bool cluster_clear(const ColConst& K, const Grid& g, const float* vals, float4 cl) {
  const float lx = __fmaf_rn(K.r[0], cl.x, __fmaf_rn(K.r[1], cl.y, __fmaf_rn(K.r[2], cl.z, K.t[0])));
  const float ly = __fmaf_rn(K.r[3], cl.x, __fmaf_rn(K.r[4], cl.y, __fmaf_rn(K.r[5], cl.z, K.t[1])));
  const float lz = __fmaf_rn(K.r[6], cl.x, __fmaf_rn(K.r[7], cl.y, __fmaf_rn(K.r[8], cl.z, K.t[2])));
  const float l1 = (fabsf(cl.x) + fabsf(cl.y) + fabsf(cl.z)) * (1.0f + 1e-6f);
  const float delta = __fmaf_rn(1e-6f, l1, K.d0);
  const float reach = (cl.w + delta) * (1.0f + 1e-6f);
  const float e = fmaxf(fmaxf(fabsf(lx - K.cx[0]) - K.hx[0], fabsf(ly - K.cx[1]) - K.hx[1]),
                        fabsf(lz - K.cx[2]) - K.hx[2]);
  if (e > reach) return true;  // every point outside the box
  // Centre clamped to the box, FP32 trilinear there, Lipschitz bound.
  const float px = fminf(fmaxf(lx, K.cx[0] - K.hx[0]), K.cx[0] + K.hx[0]);
  const float py = fminf(fmaxf(ly, K.cx[1] - K.hx[1]), K.cx[1] + K.hx[1]);
  const float pz = fminf(fmaxf(lz, K.cx[2] - K.hx[2]), K.cx[2] + K.hx[2]);
  const float v = tri32(g, vals, fmaxf(px - K.lo[0], 0.0f) * K.inv_vox, fmaxf(py - K.lo[1], 0.0f) * K.inv_vox,
                        fmaxf(pz - K.lo[2], 0.0f) * K.inv_vox);
  const float bound = v + K.vm_c + K.lip * (1.7320512f * cl.w + 3.0f * delta);
  return bound + 1e-6f * fabsf(bound) <= K.tol_dn;
}

__global__ void __launch_bounds__(kColThreads, 8) collide_kernel(DevProblem P, DevState S, int all, int count_only) {
  pdl_enter();
  const int j = blockIdx.x;
  if (!all && !S.active[j]) return;
  extern __shared__ __align__(16) unsigned int col_smem[];
  const int nwords = (P.n_scene + 31) / 32;
  const int ncl = P.n_clusters;
  unsigned int* hitbits = col_smem;                                      // bit per scene point (original order)
  // Cluster lists in shared memory, or (scenes beyond ~270k points) in the
  // particle's global scratch.
  int* list1 = P.col_lists_global ? S.col_lists + static_cast<int64_t>(j) * ncl * (1 + kSubPerCluster)
                                  : reinterpret_cast<int*>(col_smem + round_up(nwords, 4));  // left after level 1
  int* list2 = list1 + ncl;                                              // sub-clusters left after level 2
  __shared__ ColConst K;
  __shared__ int s_n1, s_n2;
  __shared__ int scan_w[kColWarps];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int pre = P.part_pre[j];
  const Grid& g = P.grids[P.pre_sdf[pre]];
  const double* th = th_of(S.theta, j);
  for (int w = tid; w < nwords; w += kColThreads) hitbits[w] = 0u;
  if (tid == 0) {
    s_n1 = 0;
    s_n2 = 0;
  }
  // The particle's FP32 frame and margins (pose_prep_kernel).
  constexpr int kWords = sizeof(ColConst) / 4;
  static_assert(sizeof(ColConst) % 4 == 0, "ColConst is copied as words");
  if (tid < kWords) reinterpret_cast<int*>(&K)[tid] = reinterpret_cast<const int*>(S.colc + j)[tid];
  __syncthreads();
  const float* vals = P.sdf_values + g.values_offset;

  // 1-2. Cluster tests: 32-point clusters, then the 8-point sub-clusters of
  // the clusters left (both in Morton order).
  int n2;
  if (!K.cull_ok) {
    n2 = ncl * kSubPerCluster;
    for (int c = tid; c < n2; c += kColThreads) list2[c] = c;
    __syncthreads();
  } else {
    for (int c = tid; c < ncl; c += kColThreads)
      if (!cluster_clear(K, g, vals, P.clusters[c])) list1[atomicAdd(&s_n1, 1)] = c;
    __syncthreads();
    const int n1 = s_n1 * kSubPerCluster;
    for (int e = tid; e < n1; e += kColThreads) {
      const int sc = list1[e / kSubPerCluster] * kSubPerCluster + e % kSubPerCluster;
      if (!cluster_clear(K, g, vals, P.subclusters[sc])) list2[atomicAdd(&s_n2, 1)] = sc;
    }
    __syncthreads();
    n2 = s_n2;
  }

  // 3. Per-point test of the remaining sub-clusters: a warp step covers
  // 32 / kSubPts sub-clusters (one lane per point) kColU times over, with every
  // load of the step issued together (the step is a chain of dependent L1/L2
  // round trips: point -> coarse block -> trilinear nodes).
  constexpr int kPerStep = 32 / kSubPts;
  const int sy = g.dims[2], sx = g.dims[1] * g.dims[2];
  const float* coarse = P.sdf_coarse + g.coarse_offset;
  for (int e0 = wid * kColU * kPerStep; e0 < n2; e0 += kColWarps * kColU * kPerStep) {
    int orig[kColU];
    float4 p[kColU];
#pragma unroll
    for (int u = 0; u < kColU; ++u) {
      const int e = e0 + u * kPerStep + lane / kSubPts;
      const int idx = (e < n2 ? list2[e] : list2[e0]) * kSubPts + lane % kSubPts;
      orig[u] = e < n2 ? P.scene_perm[idx] : -1;
      p[u] = P.scene_s32[idx];
    }
    float d[kColU], ux[kColU], uy[kColU], uz[kColU];
    int st[kColU], base[kColU];  // st: 0 clear, 1 colliding, 2 exact test, 3 coarse + trilinear
    float cm[kColU];
#pragma unroll
    for (int u = 0; u < kColU; ++u) {
      const float lx = __fmaf_rn(K.r[0], p[u].x, __fmaf_rn(K.r[1], p[u].y, __fmaf_rn(K.r[2], p[u].z, K.t[0])));
      const float ly = __fmaf_rn(K.r[3], p[u].x, __fmaf_rn(K.r[4], p[u].y, __fmaf_rn(K.r[5], p[u].z, K.t[1])));
      const float lz = __fmaf_rn(K.r[6], p[u].x, __fmaf_rn(K.r[7], p[u].y, __fmaf_rn(K.r[8], p[u].z, K.t[2])));
      d[u] = __fmaf_rn(1e-6f, p[u].w, K.d0);
      // Signed distance outside the box along the worst axis (> 0: outside).
      const float ebox = fmaxf(fmaxf(fabsf(lx - K.cx[0]) - K.hx[0], fabsf(ly - K.cx[1]) - K.hx[1]),
                               fabsf(lz - K.cx[2]) - K.hx[2]);
      // Outside: value <= -boundary_max_abs <= contact_tolerance when cull_ok.
      st[u] = orig[u] < 0 ? 0 : (ebox > d[u] ? (K.cull_ok ? 0 : 2) : (ebox < -d[u] ? 3 : 2));
      ux[u] = (lx - K.lo[0]) * K.inv_vox;
      uy[u] = (ly - K.lo[1]) * K.inv_vox;
      uz[u] = (lz - K.lo[2]) * K.inv_vox;
      const int ix = max(min(static_cast<int>(ux[u]), g.dims[0] - 2), 0);
      const int iy = max(min(static_cast<int>(uy[u]), g.dims[1] - 2), 0);
      const int iz = max(min(static_cast<int>(uz[u]), g.dims[2] - 2), 0);
      base[u] = (ix * g.dims[1] + iy) * g.dims[2] + iz;
      // Coarse bound: the FP64 cell is within one cell of this one, and its
      // trilinear value is a convex combination of nodes the dilated block
      // max covers — below the tolerance, the point cannot collide.
      cm[u] = __ldg(coarse + ((static_cast<unsigned>(ix) >> 2) * g.cdims[1] + (static_cast<unsigned>(iy) >> 2)) *
                                 g.cdims[2] +
                    (static_cast<unsigned>(iz) >> 2));  // kCoarse = 4
    }
    // Trilinear nodes of every in-box point the coarse bound does not clear
    // (the others load cell (0, 0, 0): every load of the step stays
    // unconditional, so they are issued back to back).
    float v[kColU][8];
#pragma unroll
    for (int u = 0; u < kColU; ++u) {
      if (st[u] == 3 && cm[u] <= K.cut32) st[u] = 0;
      const float* v0 = vals + (st[u] == 3 ? base[u] : 0);
      v[u][0] = __ldg(v0);
      v[u][1] = __ldg(v0 + sx);
      v[u][2] = __ldg(v0 + 1);
      v[u][3] = __ldg(v0 + sx + 1);
      v[u][4] = __ldg(v0 + sy);
      v[u][5] = __ldg(v0 + sx + sy);
      v[u][6] = __ldg(v0 + sy + 1);
      v[u][7] = __ldg(v0 + sx + sy + 1);
    }
#pragma unroll
    for (int u = 0; u < kColU; ++u) {
      if (st[u] == 3) {
        const int ix = max(min(static_cast<int>(ux[u]), g.dims[0] - 2), 0);
        const int iy = max(min(static_cast<int>(uy[u]), g.dims[1] - 2), 0);
        const int iz = max(min(static_cast<int>(uz[u]), g.dims[2] - 2), 0);
        const float fxx = fminf(fmaxf(ux[u] - ix, 0.0f), 1.0f), fyy = fminf(fmaxf(uy[u] - iy, 0.0f), 1.0f),
                    fzz = fminf(fmaxf(uz[u] - iz, 0.0f), 1.0f);
        const float c00 = __fmaf_rn(fxx, v[u][1] - v[u][0], v[u][0]);
        const float c01 = __fmaf_rn(fxx, v[u][3] - v[u][2], v[u][2]);
        const float c10 = __fmaf_rn(fxx, v[u][5] - v[u][4], v[u][4]);
        const float c11 = __fmaf_rn(fxx, v[u][7] - v[u][6], v[u][6]);
        const float c0 = __fmaf_rn(fyy, c10 - c00, c00);
        const float c1 = __fmaf_rn(fyy, c11 - c01, c01);
        const float v32 = __fmaf_rn(fzz, c1 - c0, c0);
        const float mv = K.vm_pos * 3.0f * d[u] + K.vm_c;
        st[u] = v32 > K.tol32 + mv ? 1 : (v32 < K.tol32 - mv ? 0 : 2);
      }
    }
#pragma unroll
    for (int u = 0; u < kColU; ++u) {
      bool hit = st[u] == 1;
      if (st[u] == 2)
        hit = collide_exact(th, P.grids + P.pre_sdf[pre], P.sdf_values,
                            P.scene64 + 3 * static_cast<int64_t>(orig[u]), P.contact_tolerance);
      if (hit) atomicOr(hitbits + (orig[u] >> 5), 1u << (orig[u] & 31));
    }
  }
  __syncthreads();

  // 4. Compaction in scene order: thread t owns words [t * wpt, (t + 1) * wpt),
  // a block-wide exclusive scan of the per-thread counts gives its first slot.
  const int wpt = (nwords + kColThreads - 1) / kColThreads;
  const int w0 = min(nwords, tid * wpt), w1 = min(nwords, w0 + wpt);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(hitbits[w]);
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) scan_w[wid] = incl;
  __syncthreads();
  int base_w = 0, total = 0;
  for (int w = 0; w < kColWarps; ++w) {
    base_w += w < wid ? scan_w[w] : 0;
    total += scan_w[w];
  }
  const int64_t row = static_cast<int64_t>(j) * P.n_scene;
  if (!count_only) {
    int slot = base_w + incl - cnt;
    for (int w = w0; w < w1; ++w) {
      unsigned mask = hitbits[w];
      while (mask) {
        S.col_idx[row + slot++] = w * 32 + __ffs(mask) - 1;
        mask &= mask - 1;
      }
    }
    __syncthreads();  // col_idx of the whole particle written (block-visible)
    // Reverse-match queries, spread evenly over the threads.
    const float B = __double2float_ru(S.Bs[j]);
    const V3 c = V3{S.ctr[3 * j], S.ctr[3 * j + 1], S.ctr[3 * j + 2]};
    for (int i = tid; i < total; i += kColThreads) {
      const V3 p = load3(P.scene64, S.col_idx[row + i]);
      const float fx = __double2float_rn(p.x - c.x), fy = __double2float_rn(p.y - c.y),
                  fz = __double2float_rn(p.z - c.z);
      // |a| from the rounded components, rounded up (the window margin only
      // needs an upper bound of A).
      const float A = __fsqrt_ru(__fmaf_ru(fx, fx, __fmaf_ru(fy, fy, __fmul_ru(fz, fz)))) * (1.0f + 1e-6f);
      S.col_q[row + i] = make_float4(fx, fy, fz, nn_margin32(A, B));
    }
  }
  if (tid == 0) {
    S.n_col[j] = total;
    atomicAdd(S.stats + 14, static_cast<unsigned long long>(n2));  // sub-clusters left to the point test
  }
}

constexpr size_t kColSmemMax = 200 * 1024;

static size_t collide_smem_full(const DevProblem& P) {
  return static_cast<size_t>(round_up((P.n_scene + 31) / 32, 4)) * sizeof(unsigned int) +
         static_cast<size_t>(P.n_clusters) * (1 + kSubPerCluster) * sizeof(int);
}

bool collide_lists_global(const DevProblem& P) { return collide_smem_full(P) > kColSmemMax; }

size_t collide_smem_bytes(const DevProblem& P) {
  return P.col_lists_global ? static_cast<size_t>(round_up((P.n_scene + 31) / 32, 4)) * sizeof(unsigned int)
                            : collide_smem_full(P);
}

void collide_set_attrs() {
  cudaFuncSetAttribute(collide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kColSmemMax));
}

void launch_collide(const DevProblem& P, DevState& S, int all, int count_only, cudaStream_t st) {
  pdl_launch(collide_kernel, dim3(P.J), dim3(kColThreads), collide_smem_bytes(P), st, P, S, all, count_only);
}

}  // namespace asicp
