// Device kernels of the B200 AS-ICP solver (everything but the NN search,
// which lives in nn.cu).  Reference correspondences are cited per kernel;
// every FP64 expression follows dmath.cuh's reference order (this file is
// compiled with -fmad=false).
#include "common.cuh"
#include "gexp.cuh"
#include "mt64.cuh"

#include <cuda_runtime.h>

#include <cstdint>

namespace asicp {

// ---------------------------------------------------------------------------
// K0: per-particle RNG seeding, std::mt19937_64(seed + j) (grasp.cpp:149-151).
// ---------------------------------------------------------------------------
__global__ void seed_rng_kernel(uint64_t* state, int* mti, uint64_t seed, int J) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  mt::seed_state(state + static_cast<int64_t>(j) * mt::kN, seed + static_cast<uint64_t>(j));
  mti[j] = mt::kN;
}

// ---------------------------------------------------------------------------
// K1: pose preparation — R(q) and S_world = R s + t (apply_transform,
// geometry.cpp:68-74) in FP64, plus two FP32 forms for the NN filter:
// forward queries (x, y, z, margin) centred at the object centroid, and
// reverse candidates (-2b, |b|^2) centred at the particle's TCP in world
// (keeps |b| at gripper scale, so the certification window stays tight).
// Candidate rows are padded to a multiple of 32 with +inf.
// ---------------------------------------------------------------------------
__global__ void pose_prep_kernel(DevProblem P, DevState S, int all) {
  const int j = blockIdx.x;
  if (!all && !S.active[j]) return;
  if (!all && threadIdx.x == 0) atomicAdd(S.stats + 13, 1ull);  // active (not SGD-frozen) particle evaluations
  const int pre = P.part_pre[j];
  const double* th = th_of(S.theta, j);
  const M3 r = rotation_matrix(pose_q(th));
  const V3 t = pose_t(th);
  const int s0 = P.pre_surf_off[pre], ns = P.pre_surf_off[pre + 1] - s0;
  const int64_t o = P.part_surf_off[j];
  const V3 tcp = V3{P.pre_tcp[3 * pre], P.pre_tcp[3 * pre + 1], P.pre_tcp[3 * pre + 2]};
  const V3 c = transform(r, t, tcp);
  __shared__ double s_bmax[kNnThreads];
  double bmax = 0.0;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    const V3 w = transform(r, t, load3(P.surf64, s0 + i));
    S.S64[3 * (o + i) + 0] = w.x;
    S.S64[3 * (o + i) + 1] = w.y;
    S.S64[3 * (o + i) + 2] = w.z;
    const double ax = w.x - P.center[0], ay = w.y - P.center[1], az = w.z - P.center[2];
    const double A = sqrt(ax * ax + ay * ay + az * az);
    S.Sq32[o + i] = make_float4(__double2float_rn(ax), __double2float_rn(ay), __double2float_rn(az),
                                nn_margin(A, P.B_obj));
    const double bx = w.x - c.x, by = w.y - c.y, bz = w.z - c.z;
    const float fx = __double2float_rn(bx), fy = __double2float_rn(by), fz = __double2float_rn(bz);
    const double gx = fx, gy = fy, gz = fz;
    S.Sc32[o + i] = make_float4(-2.0f * fx, -2.0f * fy, -2.0f * fz, __double2float_rn(gx * gx + gy * gy + gz * gz));
    bmax = fmax(bmax, sqrt(bx * bx + by * by + bz * bz));
  }
  for (int i = ns + threadIdx.x; i < round_up(ns, kSub); i += blockDim.x)
    S.Sc32[o + i] = make_float4(0.0f, 0.0f, 0.0f, INFINITY);
  s_bmax[threadIdx.x] = bmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < blockDim.x; ++i) m = fmax(m, s_bmax[i]);
    S.Bs[j] = m * (1.0 + 1e-6) + 1e-12;
    S.ctr[3 * j] = c.x;
    S.ctr[3 * j + 1] = c.y;
    S.ctr[3 * j + 2] = c.z;
  }
}

// ---------------------------------------------------------------------------
// K2: collision test — colliding_points (sdf.cpp:227-243) with query(stacked)
// (sdf.cpp:220-225) and trilinear query (sdf.cpp:177-203), FP64.  Writes the
// colliding scene indices in scene order and their FP32 reverse-match queries.
// count_only: final ranking (only N_col == 0 matters, grasp.cpp:271-274).
// ---------------------------------------------------------------------------
//
// Most scene points lie far outside the gripper's grid box, where the
// reference returns -(distance + boundary_max_abs) <= -boundary_max_abs.  When
// contact_tolerance >= -boundary_max_abs such points can never collide, so an
// FP32 transform that places a point outside the box by more than a
// conservative rounding margin decides it without the FP64 path; every other
// point takes the exact FP64 evaluation.  Each warp owns a contiguous scene
// range; hits are kept as a bitmask in shared memory and compacted in scene
// order after a scan over the warps' counts.
constexpr int kColThreads = 256;
constexpr int kColWarps = kColThreads / 32;

// The exact FP64 test of one scene point (colliding_points body,
// sdf.cpp:237-239), kept out of line so its register needs do not throttle
// the FP32 pre-test loop (it runs for ~1e-4 of the points).
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

__global__ void __launch_bounds__(kColThreads, 3) collide_kernel(DevProblem P, DevState S, int all, int count_only) {
  const int j = blockIdx.x;
  if (!all && !S.active[j]) return;
  extern __shared__ __align__(16) unsigned int hitbits[];  // ceil(n_scene / 32) words, then the coarse grid
  __shared__ int warp_cnt[kColWarps];
  const int pre = P.part_pre[j];
  const Grid g = P.grids[P.pre_sdf[pre]];
  float* coarse_s = reinterpret_cast<float*>(hitbits + round_up((P.n_scene + 31) / 32, 4));
  const int ncoarse = g.cdims[0] * g.cdims[1] * g.cdims[2];
  for (int i = threadIdx.x; i < ncoarse; i += blockDim.x) coarse_s[i] = P.sdf_coarse[g.coarse_offset + i];
  const double coarse_cut = P.contact_tolerance - 1e-12 * (1.0 + fabs(P.contact_tolerance));
  __syncthreads();
  const double* th = th_of(S.theta, j);
  Q4 qi;
  V3 ti;
  inverse(pose_q(th), pose_t(th), &qi, &ti);
  const M3 r = rotation_matrix(qi);
  const V3 off = V3{g.offset[0], g.offset[1], g.offset[2]};
  // FP32 culling box (sdf.cpp:178-182 out-of-grid test) with margin.
  float r32[9];
  for (int i = 0; i < 9; ++i) r32[i] = static_cast<float>(r.m[i]);
  const float t32x = static_cast<float>(ti.x), t32y = static_cast<float>(ti.y), t32z = static_cast<float>(ti.z);
  float lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = static_cast<float>(g.origin[a]);
    hi[a] = static_cast<float>(g.origin[a] + g.voxel * static_cast<double>(g.dims[a] - 1));
  }
  const float tn = fabsf(t32x) + fabsf(t32y) + fabsf(t32z) + fabsf(lo[0]) + fabsf(lo[1]) + fabsf(lo[2]) +
                   fabsf(hi[0]) + fabsf(hi[1]) + fabsf(hi[2]);
  // Box as centre +- half extent; cbox covers the rounding of cx, hx and of
  // the |l - c| - h evaluation (a few ulps of the box coordinates).
  float cx[3], hx[3];
  for (int a = 0; a < 3; ++a) {
    cx[a] = 0.5f * (lo[a] + hi[a]);
    hx[a] = 0.5f * (hi[a] - lo[a]);
  }
  const float cbox = 1e-6f * (fabsf(lo[0]) + fabsf(lo[1]) + fabsf(lo[2]) + fabsf(hi[0]) + fabsf(hi[1]) + fabsf(hi[2]));
  const float d0 = 1e-6f * (1.0f + tn) + cbox;
  // Largest float below coarse_cut: cm < coarse_cut  <=>  cm <= cut32.
  float cut32 = static_cast<float>(coarse_cut);
  if (static_cast<double>(cut32) >= coarse_cut) cut32 = nextafterf(cut32, -INFINITY);
  const bool cull_ok = P.contact_tolerance >= -g.boundary_max_abs;
  const float inv_vox = static_cast<float>(1.0 / g.voxel);
  const float tol32 = static_cast<float>(P.contact_tolerance);
  // Value margin: slope x position error, plus fraction rounding (|u| <= dims,
  // ~1e-5 voxel) and 7 FP32 lerps / the rounded tolerance (~1e-6 x magnitudes).
  const float vmargin_pos = static_cast<float>(g.lip);
  const float vmargin_c = static_cast<float>(g.lip * g.voxel * 1e-5 + 1e-6 * (g.vmax + fabs(P.contact_tolerance)) +
                                             1e-9);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwords = (P.n_scene + 31) / 32;
  const int words_per_warp = (nwords + kColWarps - 1) / kColWarps;
  const int w0 = wid * words_per_warp, w1 = min(nwords, w0 + words_per_warp);
  int cnt = 0;
  // Status per point: 0 clear, 1 colliding, 2 needs the exact FP64 test.
  auto classify = [&](float4 p) -> int {
    int status = 2;
    {
      {
        const float fx = p.x, fy = p.y, fz = p.z;
        const float lx = __fmaf_rn(r32[0], fx, __fmaf_rn(r32[1], fy, __fmaf_rn(r32[2], fz, t32x)));
        const float ly = __fmaf_rn(r32[3], fx, __fmaf_rn(r32[4], fy, __fmaf_rn(r32[5], fz, t32y)));
        const float lz = __fmaf_rn(r32[6], fx, __fmaf_rn(r32[7], fy, __fmaf_rn(r32[8], fz, t32z)));
        // |l32 - l64| <= ~5u (|p|_1 + |t|_1) (+ the rounded box corners): d is
        // >= 3x that (p.w = |p|_1, prepared on the host).
        const float d = __fmaf_rn(1e-6f, p.w, d0);
        // Signed distance outside the box along the worst axis (> 0: outside).
        const float e = fmaxf(fmaxf(fabsf(lx - cx[0]) - hx[0], fabsf(ly - cx[1]) - hx[1]), fabsf(lz - cx[2]) - hx[2]);
        const bool out_far = e > d;
        const bool in_far = e < -d;
        if (out_far) {
          if (cull_ok) status = 0;  // value <= -boundary_max_abs <= contact_tolerance: never collides
        } else if (in_far) {
          // FP32 trilinear; the interpolant is continuous with per-axis slope
          // <= lip, so |v32 - v64| <= lip * (|e|_1 + fraction error) + lerp rounding.
          const float ux = (lx - lo[0]) * inv_vox, uy = (ly - lo[1]) * inv_vox, uz = (lz - lo[2]) * inv_vox;
          const int ix = max(min(static_cast<int>(ux), g.dims[0] - 2), 0);
          const int iy = max(min(static_cast<int>(uy), g.dims[1] - 2), 0);
          const int iz = max(min(static_cast<int>(uz), g.dims[2] - 2), 0);
          // Coarse bound: the FP64 cell is within one cell of this one, and its
          // trilinear value is a convex combination of nodes the dilated block
          // max covers — below the tolerance, the point cannot collide.
          const float cm = coarse_s[((static_cast<unsigned>(ix) >> 2) * g.cdims[1] + (static_cast<unsigned>(iy) >> 2)) *
                                        g.cdims[2] +
                                    (static_cast<unsigned>(iz) >> 2)];  // kCoarse = 4
          if (cm <= cut32) return 0;
          const float fxx = fminf(fmaxf(ux - ix, 0.0f), 1.0f), fyy = fminf(fmaxf(uy - iy, 0.0f), 1.0f),
                      fzz = fminf(fmaxf(uz - iz, 0.0f), 1.0f);
          const float* v0 = P.sdf_values + g.values_offset + (static_cast<int64_t>(ix) * g.dims[1] + iy) * g.dims[2] + iz;
          const int sy = g.dims[2], sx = g.dims[1] * g.dims[2];
          const float c00 = __fmaf_rn(fxx, v0[sx] - v0[0], v0[0]);
          const float c01 = __fmaf_rn(fxx, v0[sx + 1] - v0[1], v0[1]);
          const float c10 = __fmaf_rn(fxx, v0[sx + sy] - v0[sy], v0[sy]);
          const float c11 = __fmaf_rn(fxx, v0[sx + sy + 1] - v0[sy + 1], v0[sy + 1]);
          const float c0 = __fmaf_rn(fyy, c10 - c00, c00);
          const float c1 = __fmaf_rn(fyy, c11 - c01, c01);
          const float v32 = __fmaf_rn(fzz, c1 - c0, c0);
          const float mv = vmargin_pos * 3.0f * d + vmargin_c;
          if (v32 > tol32 + mv)
            status = 1;
          else if (v32 < tol32 - mv)
            status = 0;
        }
      }
    }
    return status;
  };
  constexpr int kU = 4;  // words per batch: independent loads in flight
  for (int wb = w0; wb < w1; wb += kU) {
    float4 pv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = (wb + u) * 32 + lane;
      pv[u] = (wb + u < w1 && idx < P.n_scene) ? P.scene32[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    int stt[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = (wb + u) * 32 + lane;
      stt[u] = (wb + u < w1 && idx < P.n_scene) ? classify(pv[u]) : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (wb + u >= w1) break;
      bool hit = stt[u] == 1;
      if (stt[u] == 2)
        hit = collide_exact(th, P.grids + P.pre_sdf[pre], P.sdf_values,
                            P.scene64 + 3 * static_cast<int64_t>((wb + u) * 32 + lane), P.contact_tolerance);
      const unsigned mask = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) hitbits[wb + u] = mask;
      cnt += __popc(mask);
    }
  }
  if (lane == 0) warp_cnt[wid] = cnt;
  __syncthreads();
  int base = 0, total = 0;
  for (int w = 0; w < kColWarps; ++w) {
    base += w < wid ? warp_cnt[w] : 0;
    total += warp_cnt[w];
  }
  if (!count_only && cnt > 0) {
    const int64_t row = static_cast<int64_t>(j) * P.n_scene;
    const double B = S.Bs[j];
    const V3 c = V3{S.ctr[3 * j], S.ctr[3 * j + 1], S.ctr[3 * j + 2]};
    for (int w = w0; w < w1; ++w) {
      const unsigned mask = hitbits[w];
      if (mask == 0) continue;
      if ((mask >> lane) & 1u) {
        const int idx = w * 32 + lane;
        const int slot = base + __popc(mask & ((1u << lane) - 1u));
        S.col_idx[row + slot] = idx;
        const V3 p = load3(P.scene64, idx);
        const double ax = p.x - c.x, ay = p.y - c.y, az = p.z - c.z;
        const double A = sqrt(ax * ax + ay * ay + az * az);
        S.col_q[row + slot] =
            make_float4(__double2float_rn(ax), __double2float_rn(ay), __double2float_rn(az), nn_margin(A, B));
      }
      base += __popc(mask);
    }
  }
  if (threadIdx.x == 0) S.n_col[j] = total;
}

// ---------------------------------------------------------------------------
// K5: minibatch sampling — sample_minibatch / sample_minibatch_indices
// (spatial_index.cpp:111-131) with Rng::uniform_index (rng.hpp:32-44) on the
// particle's own mt19937_64 stream.  Only non-colliding active particles
// draw (grasp.cpp:183-184).  Output: pool object indices in sample order and
// the gathered FP32 candidates (+inf padded to a multiple of 32).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t serial_next(uint64_t* st, int* mti) {
  if (*mti >= mt::kN) {
    mt::twist_serial(st);
    *mti = 0;
  }
  return mt::temper(st[(*mti)++]);
}

template <bool kSmemIdx>
__global__ void __launch_bounds__(128) minibatch_kernel(DevProblem P, DevState S, int m) {
  const int j = blockIdx.x;
  if (!S.active[j] || S.n_col[j] > 0) return;
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ uint64_t st[mt::kN];
  __shared__ uint64_t outs[mt::kN];
  __shared__ uint32_t jbuf[mt::kN];
  __shared__ int s_mti, s_reject;
  const int n = P.n_obj;
  int* idx = kSmemIdx ? reinterpret_cast<int*>(dyn) : S.fy_scratch + static_cast<int64_t>(j) * n;
  int* pool = S.pool_idx + static_cast<int64_t>(j) * P.n_obj_pad;
  uint64_t* gst = S.rng_state + static_cast<int64_t>(j) * mt::kN;
  for (int i = threadIdx.x; i < mt::kN; i += blockDim.x) st[i] = gst[i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) idx[i] = i;  // iota (spatial_index.cpp:115-116)
  if (threadIdx.x == 0) s_mti = S.rng_mti[j];
  __syncthreads();
  int i0 = 0;
  while (i0 < m) {
    if (s_mti >= mt::kN) {
      mt::twist_block(st);
      if (threadIdx.x == 0) s_mti = 0;
      __syncthreads();
    }
    const int mti = s_mti;
    const int cnt = min(mt::kN - mti, m - i0);
    for (int t = threadIdx.x; t < mt::kN; t += blockDim.x) outs[t] = mt::temper(st[t]);
    if (threadIdx.x == 0) s_reject = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      uint64_t u;
      const uint64_t range = static_cast<uint64_t>(n - (i0 + t));
      if (!mt::lemire(outs[mti + t], range, &u)) s_reject = 1;
      jbuf[t] = static_cast<uint32_t>(i0 + t + u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int consumed = cnt;
      int done = cnt;
      if (s_reject) {
        // Rare rejection (probability ~n/2^64 per draw): redo this block
        // serially so the engine consumes exactly what the reference does.
        int lm = mti;
        done = 0;
        while (done < cnt && lm < mt::kN) {
          const uint64_t range = static_cast<uint64_t>(n - (i0 + done));
          uint64_t u;
          uint64_t x = mt::temper(st[lm++]);
          while (!mt::lemire(x, range, &u)) x = serial_next(st, &lm);
          jbuf[done] = static_cast<uint32_t>(i0 + done + u);
          ++done;
        }
        consumed = -1;
        s_mti = lm;
      }
      // Partial Fisher-Yates swaps (spatial_index.cpp:117-120).  Position i
      // is final after step i, so its value goes straight to the pool.
      for (int t = 0; t < done; ++t) {
        const int i = i0 + t;
        const int jj = static_cast<int>(jbuf[t]);
        const int a = idx[i];
        const int b = idx[jj];
        idx[jj] = a;
        pool[i] = b;
      }
      if (consumed >= 0) s_mti = mti + consumed;
      jbuf[0] = static_cast<uint32_t>(done);
    }
    __syncthreads();
    i0 += static_cast<int>(jbuf[0]);
    __syncthreads();
  }
  for (int i = threadIdx.x; i < mt::kN; i += blockDim.x) gst[i] = st[i];
  if (threadIdx.x == 0) S.rng_mti[j] = s_mti;
  __syncthreads();
  float4* pool32 = S.pool32 + static_cast<int64_t>(j) * P.n_obj_pad;  // pair-interleaved (pc_*)
  gather_pool(P.obj_cand4, pool, m, pool32, threadIdx.x, blockDim.x);
}

// ---------------------------------------------------------------------------
// K4: cost / gradient — grasp_gradients + contact_loss + com_loss
// (grasp.cpp:37-66) for the forward branch, collision_loss_and_gradients +
// sgd_icp_gradients (grasp.cpp:68-84, optim.cpp:92-106) for the colliding
// branch.  Per-pair terms are computed in parallel; the 8 running sums are
// accumulated in pair order by 8 threads, exactly like the reference loops.
// ---------------------------------------------------------------------------
constexpr int kCostThreads = 256;           // two particles per CTA, 128 threads each
constexpr int kCostHalf = 128;
constexpr int kCostChunk = 512;              // pairs per chunk and particle
constexpr int kCostRow = kCostChunk + 1;     // +1 double: the 8 summing threads hit distinct banks
constexpr int kCostSmem = 2 * 8 * kCostRow * 8;  // bytes (both halves)

// Each half of the CTA (128 threads, its own named barrier) owns one particle:
// 384 CTAs of 2 x 32 KB of terms fit one wave at 3 CTAs/SM, where one
// particle per CTA took two.
__global__ void __launch_bounds__(kCostThreads) cost_kernel(DevProblem P, DevState S, int final_pass) {
  const int half = threadIdx.x >= kCostHalf ? 1 : 0;
  const int tid = threadIdx.x - half * kCostHalf;
  const int j = 2 * blockIdx.x + half;
  if (j >= P.J) return;
  if (!final_pass && !S.active[j]) return;
  extern __shared__ double cost_smem[];
  double* cost_terms = cost_smem + half * 8 * kCostRow;  // [8][kCostRow]
  __shared__ double acc2[2][8];
  double* acc = acc2[half];
  auto half_sync = [half]() {
    if (half)
      asm volatile("bar.sync 2, %0;" ::"n"(kCostHalf) : "memory");
    else
      asm volatile("bar.sync 1, %0;" ::"n"(kCostHalf) : "memory");
  };
  const int pre = P.part_pre[j];
  const double* th = th_of(S.theta, j);
  const Q4 q = pose_q(th);
  const V3 t = pose_t(th);
  const M3 r = rotation_matrix(q);
  M3 dR[4];
  rotation_matrix_derivatives(q, dR);
  const int s0 = P.pre_surf_off[pre];
  const int64_t so = P.part_surf_off[j];
  const int ns = P.pre_surf_off[pre + 1] - s0;
  const bool reverse = !final_pass && S.n_col[j] > 0;
  const int npairs = reverse ? S.n_col[j] : ns;
  const V3 tcp = V3{P.pre_tcp[3 * pre], P.pre_tcp[3 * pre + 1], P.pre_tcp[3 * pre + 2]};
  const V3 com = V3{P.com[0], P.com[1], P.com[2]};
  const V3 com_residual = sub(add(mul(r, tcp), t), com);
  if (tid < 8) {
    double init = 0.0;
    if (!reverse) {
      if (tid < 3)
        init = tid == 0 ? com_residual.x : (tid == 1 ? com_residual.y : com_residual.z);
      else if (tid < 7)
        init = dot(com_residual, mul(dR[tid - 3], tcp));
    }
    acc[tid] = init;  // slot 7: contact-loss sum starts at 0.0
  }
  const int64_t row = static_cast<int64_t>(j) * P.n_scene;
  const int* pmap = final_pass ? nullptr : S.pool_map;
  for (int c0 = 0; c0 < npairs; c0 += kCostChunk) {
    const int n = min(kCostChunk, npairs - c0);
    for (int e = tid; e < n; e += kCostHalf) {
      const int i = c0 + e;
      V3 src, tr, ref;
      if (reverse) {
        const int sidx = S.res_rev[row + i];
        src = load3(P.surf64, s0 + sidx);
        tr = load3(S.S64, so + sidx);
        ref = load3(P.scene64, S.col_idx[row + i]);
      } else {
        src = load3(P.surf64, s0 + i);
        tr = load3(S.S64, so + i);
        const int pos = S.res_fwd[so + i];
        const int64_t oi = pmap ? pmap[static_cast<int64_t>(j) * P.n_obj_pad + pos] : pos;
        ref = load3(P.obj64, oi);
      }
      const V3 res = sub(tr, ref);
      cost_terms[0 * kCostRow + e] = res.x;
      cost_terms[1 * kCostRow + e] = res.y;
      cost_terms[2 * kCostRow + e] = res.z;
      for (int jj = 0; jj < 4; ++jj) cost_terms[(3 + jj) * kCostRow + e] = dot(res, mul(dR[jj], src));
      cost_terms[7 * kCostRow + e] = sqnorm(res);
    }
    half_sync();
    if (tid < 8) {
      // The reference's running sums, in pair order (the critical path).
      const double* tr = cost_terms + tid * kCostRow;
      double a = acc[tid];
#pragma unroll 8
      for (int e = 0; e < n; ++e) a = a + tr[e];
      acc[tid] = a;
    }
    half_sync();
  }
  if (tid == 0) {
    const double m = static_cast<double>(npairs);
    const double contact = acc[7] / m;
    const double loss = reverse ? contact : contact + sqnorm(com_residual);  // total_loss(contact, com_loss)
    if (final_pass) {
      S.final_loss[j] = loss;
      S.final_free[j] = S.n_col[j] == 0 ? 1 : 0;
      return;
    }
    double* g = S.grad + 7 * j;
    for (int a = 0; a < 7; ++a) g[a] = acc[a] / m;
    S.loss[j] = loss;
    S.in_col[j] = reverse ? 1 : 0;
    // prior_log_gradient (optim.cpp:146-156)
    double* pg = S.prior + 7 * j;
    for (int a = 0; a < 3; ++a) {
      const double var = P.prior_t_sigma[a] * P.prior_t_sigma[a];
      pg[a] = -(th[a] - P.prior_t_mean[a]) / var;
    }
    for (int a = 0; a < 4; ++a) pg[3 + a] = -P.prior_q_kappa[a] * sin(th[3 + a] - P.prior_q_location[a]);
  }
}

// ---------------------------------------------------------------------------
// Trace (grasp.cpp:197-209): pre-update pose, loss, collision flag.
// ---------------------------------------------------------------------------
__global__ void trace_kernel(DevProblem P, DevState S, int k) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.J) return;
  const int64_t r = static_cast<int64_t>(k) * P.J + j;
  for (int a = 0; a < 7; ++a) S.trace_theta[7 * r + a] = S.theta[7 * j + a];
  S.trace_loss[r] = S.loss[j];
  S.trace_col[r] = S.in_col[j];
}

// ---------------------------------------------------------------------------
// K6: SVGD.  drift = gamma (n_ref g + prior) (optim.cpp:174-178);
// h = max(median_{i<j} |t_i - t_j|^2 / log(K+1), 1e-6) (optim.cpp:133-144) by an
// exact radix select on the FP64 bit patterns; direction (optim.cpp:180-223)
// summed over i in order; update (optim.cpp:225-237).
// ---------------------------------------------------------------------------
__global__ void drift_kernel(DevProblem P, DevState S, double gamma, double n_ref) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.J) return;
  for (int a = 0; a < 7; ++a) S.drift[7 * j + a] = gamma * (n_ref * S.grad[7 * j + a] + S.prior[7 * j + a]);
}

// Small populations: median_kernel in median.cu.

// Large populations (K >= kMedBigK, e.g. cfg5's 16384 particles: 134M pair
// keys): the same exact radix select spread over the whole GPU.  Six passes
// of 12/12/12/12/12/4 bits; every pass recomputes the keys tile by tile
// (128 x 128 blocks of the upper triangle, partner poses in shared memory —
// FP64 math is cheaper than re-reading a cached 1 GB key array), counts the
// keys matching the selected prefix into a per-CTA shared histogram with
// warp-aggregated atomics, and flushes it to a global histogram; a one-CTA
// select kernel then picks the digit holding rank M/2.  The key multiset and
// the order statistic are those of the single-CTA kernel.
constexpr int kMedTile = 128;
constexpr int kMedBins = 4096;

__device__ __forceinline__ bool med_big(const DevProblem& P, int pop, int& b, int& K) {
  if (P.pop_off[pop + 1] == P.pop_off[pop] || P.bandwidth_mode == 1) return false;
  b = P.gpop_off[pop];
  K = P.gpop_off[pop + 1] - b;
  return K >= kMedBigK;
}

__global__ void med_init_kernel(DevProblem P, DevState S) {
  const int pop = blockIdx.x;
  int b, K;
  if (!med_big(P, pop, b, K)) return;
  for (int i = threadIdx.x; i < kMedBins; i += blockDim.x) S.med_hist[pop * kMedBins + i] = 0;
  if (threadIdx.x == 0) {
    MedState& m = S.med_state[pop];
    m.prefix = 0;
    m.mask = 0;
    m.rank = static_cast<long long>(K) * (K - 1) / 2 / 2;
  }
}

__global__ void __launch_bounds__(256) med_hist_kernel(DevProblem P, DevState S, int shift, int bits) {
  const int pop = blockIdx.y;
  int b, K;
  if (!med_big(P, pop, b, K)) return;
  __shared__ unsigned int hist[kMedBins];
  __shared__ double ta[kMedTile][3], tb[kMedTile][3];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < kMedBins; i += blockDim.x) hist[i] = 0;
  const unsigned long long prefix = S.med_state[pop].prefix, mask = S.med_state[pop].mask;
  const unsigned int dmask = (1u << bits) - 1u;
  const int nb = (K + kMedTile - 1) / kMedTile;
  const long long tiles = static_cast<long long>(nb) * (nb + 1) / 2;
  for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    int bi = 0;
    long long rem = tile;
    while (rem >= nb - bi) {
      rem -= nb - bi;
      ++bi;
    }
    const int bj = bi + static_cast<int>(rem);
    const int ni = min(kMedTile, K - bi * kMedTile), nj = min(kMedTile, K - bj * kMedTile);
    __syncthreads();
    for (int e = tid; e < kMedTile * 3; e += blockDim.x) {
      const int r = e / 3, a = e % 3;
      ta[r][a] = r < ni ? S.theta_all[7 * (b + bi * kMedTile + r) + a] : 0.0;
      tb[r][a] = r < nj ? S.theta_all[7 * (b + bj * kMedTile + r) + a] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < kMedTile * kMedTile; e += blockDim.x) {  // uniform trip count per warp
      const int ii = e / kMedTile, jj = e % kMedTile;
      bool hit = ii < ni && jj < nj && (bi < bj || ii < jj);
      unsigned int digit = 0;
      if (hit) {
        const double d2 = sqnorm(sub(V3{ta[ii][0], ta[ii][1], ta[ii][2]}, V3{tb[jj][0], tb[jj][1], tb[jj][2]}));
        const unsigned long long key = static_cast<unsigned long long>(__double_as_longlong(d2));
        hit = (key & mask) == prefix;
        digit = static_cast<unsigned int>(key >> shift) & dmask;
      }
      const unsigned int active = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const unsigned int peers = __match_any_sync(active, digit);
        if (__ffs(peers) - 1 == lane) atomicAdd(&hist[digit], static_cast<unsigned int>(__popc(peers)));
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < kMedBins; i += blockDim.x)
    if (hist[i]) atomicAdd(&S.med_hist[pop * kMedBins + i], hist[i]);
}

__global__ void __launch_bounds__(1024) med_select_kernel(DevProblem P, DevState S, int shift, int bits,
                                                          int last) {
  const int pop = blockIdx.x;
  int b, K;
  if (!med_big(P, pop, b, K)) return;
  unsigned int* hist = S.med_hist + pop * kMedBins;
  const int nbins = 1 << bits;
  constexpr int kPer = kMedBins / 1024;
  __shared__ long long part[1024];
  __shared__ int s_digit;
  __shared__ long long s_below;
  const int tid = threadIdx.x;
  long long mine = 0;
  for (int k = 0; k < kPer; ++k) {
    const int bin = tid * kPer + k;
    if (bin < nbins) mine += hist[bin];
  }
  part[tid] = mine;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive scan
    const long long v = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  const long long rank = S.med_state[pop].rank;
  const long long before = tid ? part[tid - 1] : 0;
  if (rank >= before && rank < part[tid]) {
    long long acc = before;
    for (int k = 0; k < kPer; ++k) {
      const int bin = tid * kPer + k;
      const long long c = bin < nbins ? hist[bin] : 0;
      if (rank < acc + c) {
        s_digit = bin;
        s_below = acc;
        break;
      }
      acc += c;
    }
  }
  __syncthreads();
  for (int i = tid; i < kMedBins; i += blockDim.x) hist[i] = 0;
  if (tid == 0) {
    MedState& m = S.med_state[pop];
    m.rank = rank - s_below;
    m.prefix |= static_cast<unsigned long long>(s_digit) << shift;
    m.mask |= static_cast<unsigned long long>(nbins - 1) << shift;
    if (last) {
      const double median = __longlong_as_double(static_cast<long long>(m.prefix));
      const double h = median / P.pop_logk1[pop];
      S.h[pop] = h < 1e-6 ? 1e-6 : h;  // std::max(h, 1e-6)
    }
  }
}

// Stein direction + update.  CTA = (population, block of 32 particles j).
// For each 32-wide tile of partners i the CTA evaluates the 32x32 kernel
// values once (glibc-exact exp) into shared memory; then 7 threads per j (one
// per pose component) accumulate their component over i in order — the
// reference's per-component left-to-right sums.
constexpr int kSvgdJ = 32;
__global__ void __launch_bounds__(kSvgdJ * 7) svgd_kernel(DevProblem P, DevState S, double eta) {
  const int pop = blockIdx.y;
  const int lb = P.pop_off[pop], Kl = P.pop_off[pop + 1] - lb;  // own (local) rows
  const int b = P.gpop_off[pop], K = P.gpop_off[pop + 1] - b;   // partners (global)
  const int j0 = blockIdx.x * kSvgdJ;
  if (j0 >= Kl) return;
  const int own0 = P.j_lo + lb - b;  // position of local row lb within the population
  __shared__ double kv[kSvgdJ][kSvgdJ + 1];   // rbf value [i][j]
  __shared__ double kq[kSvgdJ][kSvgdJ + 1];   // |q_i . q_j|
  __shared__ double ti[kSvgdJ][7];            // partner poses
  __shared__ double di[kSvgdJ][7];            // partner drifts
  __shared__ double tj[kSvgdJ][7];            // own poses
  __shared__ double dir[kSvgdJ][7];
  const int tid = threadIdx.x;
  const int jl = tid / 7, comp = tid % 7;
  const int nj = min(kSvgdJ, Kl - j0);
  for (int e = tid; e < nj * 7; e += blockDim.x) tj[e / 7][e % 7] = S.theta[7 * (lb + j0 + e / 7) + e % 7];
  const double h = S.h[pop];
  const double two_h = 2.0 / h;
  double acc = 0.0;
  for (int i0 = 0; i0 < K; i0 += kSvgdJ) {
    const int ni = min(kSvgdJ, K - i0);
    __syncthreads();
    for (int e = tid; e < ni * 7; e += blockDim.x) {
      ti[e / 7][e % 7] = S.theta_all[7 * (b + i0 + e / 7) + e % 7];
      di[e / 7][e % 7] = S.drift_all[7 * (b + i0 + e / 7) + e % 7];
    }
    __syncthreads();
    for (int e = tid; e < ni * nj; e += blockDim.x) {
      const int ii = e / nj, jj = e % nj;
      const V3 a = V3{ti[ii][0], ti[ii][1], ti[ii][2]};
      const V3 c = V3{tj[jj][0], tj[jj][1], tj[jj][2]};
      kv[ii][jj] = glibc_exp(-sqnorm(sub(a, c)) / h);  // rbf_kernel (optim.cpp:120-125)
      const double dq = ((ti[ii][3] * tj[jj][3] + ti[ii][4] * tj[jj][4]) + ti[ii][5] * tj[jj][5]) +
                        ti[ii][6] * tj[jj][6];
      kq[ii][jj] = fabs(dq);  // rotation_kernel (optim.cpp:127-131)
    }
    __syncthreads();
    if (jl < nj) {
      const int jg = own0 + j0 + jl;
      for (int ii = 0; ii < ni; ++ii) {
        const double d = di[ii][comp];
        if (i0 + ii == jg) {
          acc = acc - d;  // analytic self-term (optim.cpp:206-212)
        } else if (comp < 3) {
          const double v = kv[ii][jl];
          acc = acc + (-d) * v;
          acc = acc + (two_h * (tj[jl][comp] - ti[ii][comp])) * v;
        } else {
          acc = acc + (-d) * kq[ii][jl];
        }
      }
    }
  }
  if (jl < nj) dir[jl][comp] = acc;
  __syncthreads();
  if (tid < nj) {
    double* out = S.theta_next + 7 * (lb + j0 + tid);
    for (int a = 0; a < 3; ++a) out[a] = tj[tid][a] + eta * dir[tid][a];
    const Q4 qn = normalized(Q4{tj[tid][3] + eta * dir[tid][3], tj[tid][4] + eta * dir[tid][4],
                                tj[tid][5] + eta * dir[tid][5], tj[tid][6] + eta * dir[tid][6]});
    out[3] = qn.w;
    out[4] = qn.x;
    out[5] = qn.y;
    out[6] = qn.z;
  }
}

// Split form for small populations (the fused kernel above has only K/32
// CTAs per population): (1) every (partner i, own j) kernel value pair
// (rbf, |q_i . q_j|) in a grid of 32 x 32 tiles, into S.kmat; (2) the ordered
// accumulation — one warp per pose component, one lane per own particle, the
// same left-to-right sums and update as svgd_kernel.
__global__ void __launch_bounds__(256) svgd_kmat_kernel(DevProblem P, DevState S) {
  const int pop = blockIdx.z;
  const int lb = P.pop_off[pop], Kl = P.pop_off[pop + 1] - lb;
  const int b = P.gpop_off[pop], K = P.gpop_off[pop + 1] - b;
  const int j0 = blockIdx.x * kSvgdJ, i0 = blockIdx.y * kSvgdJ;
  if (j0 >= Kl || i0 >= K) return;
  __shared__ double ti[kSvgdJ][7], tj[kSvgdJ][7];
  const int nj = min(kSvgdJ, Kl - j0), ni = min(kSvgdJ, K - i0);
  for (int e = threadIdx.x; e < kSvgdJ * 7; e += blockDim.x) {
    const int r = e / 7, a = e % 7;
    ti[r][a] = r < ni ? S.theta_all[7 * (b + i0 + r) + a] : 0.0;
    tj[r][a] = r < nj ? S.theta[7 * (lb + j0 + r) + a] : 0.0;
  }
  __syncthreads();
  const double h = S.h[pop];
  double2* km = S.kmat + P.kofs[pop];
  for (int e = threadIdx.x; e < kSvgdJ * kSvgdJ; e += blockDim.x) {
    const int ii = e / kSvgdJ, jj = e % kSvgdJ;
    if (ii >= ni || jj >= nj) continue;
    const V3 a = V3{ti[ii][0], ti[ii][1], ti[ii][2]};
    const V3 c = V3{tj[jj][0], tj[jj][1], tj[jj][2]};
    const double kv = glibc_exp(-sqnorm(sub(a, c)) / h);  // rbf_kernel (optim.cpp:120-125)
    const double dq = ((ti[ii][3] * tj[jj][3] + ti[ii][4] * tj[jj][4]) + ti[ii][5] * tj[jj][5]) +
                      ti[ii][6] * tj[jj][6];
    km[static_cast<int64_t>(i0 + ii) * Kl + j0 + jj] = make_double2(kv, fabs(dq));  // rotation_kernel (:127-131)
  }
}

__global__ void __launch_bounds__(kSvgdJ * 7) svgd_acc_kernel(DevProblem P, DevState S, double eta) {
  const int pop = blockIdx.y;
  const int lb = P.pop_off[pop], Kl = P.pop_off[pop + 1] - lb;
  const int b = P.gpop_off[pop], K = P.gpop_off[pop + 1] - b;
  const int j0 = blockIdx.x * kSvgdJ;
  if (j0 >= Kl) return;
  __shared__ double dir[kSvgdJ][7];
  __shared__ double2 kt[kSvgdJ][kSvgdJ];  // [partner][own] of the current 32-partner tile
  __shared__ double dt[kSvgdJ][7], tt[kSvgdJ][7];
  constexpr int kT = kSvgdJ * 7;
  constexpr int kPer = (kSvgdJ * kSvgdJ + kT - 1) / kT;
  const int tid = threadIdx.x;
  const int comp = tid / 32, jl = tid % 32;
  const int nj = min(kSvgdJ, Kl - j0);
  const int jg = P.j_lo + lb - b + j0 + jl;  // own position within the population
  const double two_h = 2.0 / S.h[pop];
  const double own = jl < nj ? S.theta[7 * (lb + j0 + jl) + comp] : 0.0;
  const double2* km = S.kmat + P.kofs[pop];
  // The next tile is fetched into registers while the current one is summed.
  double2 rk[kPer];
  double rd = 0.0, rt = 0.0;
  auto fetch = [&](int i0) {
    const int ni = min(kSvgdJ, K - i0);
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kT, ii = e / kSvgdJ, jj = e % kSvgdJ;
      rk[u] = (e < kSvgdJ * kSvgdJ && ii < ni && jj < nj) ? km[static_cast<int64_t>(i0 + ii) * Kl + j0 + jj]
                                                          : make_double2(0.0, 0.0);
    }
    const int r = tid / 7, a = tid % 7;
    rd = r < ni ? S.drift_all[7 * (b + i0 + r) + a] : 0.0;
    rt = r < ni ? S.theta_all[7 * (b + i0 + r) + a] : 0.0;
  };
  fetch(0);
  double acc = 0.0;
  for (int i0 = 0; i0 < K; i0 += kSvgdJ) {
    __syncthreads();  // the previous tile is consumed
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kT;
      if (e < kSvgdJ * kSvgdJ) kt[e / kSvgdJ][e % kSvgdJ] = rk[u];
    }
    dt[tid / 7][tid % 7] = rd;
    tt[tid / 7][tid % 7] = rt;
    __syncthreads();
    if (i0 + kSvgdJ < K) fetch(i0 + kSvgdJ);
    const int ni = min(kSvgdJ, K - i0);
    for (int ii = 0; ii < ni; ++ii) {
      const double d = dt[ii][comp];
      if (i0 + ii == jg) {
        acc = acc - d;  // analytic self-term (optim.cpp:206-212)
      } else if (comp < 3) {
        const double v = kt[ii][jl].x;
        acc = acc + (-d) * v;
        acc = acc + (two_h * (own - tt[ii][comp])) * v;
      } else {
        acc = acc + (-d) * kt[ii][jl].y;
      }
    }
  }
  if (jl < nj) dir[jl][comp] = acc;
  __syncthreads();
  if (threadIdx.x < nj) {
    const int j = threadIdx.x;
    const double* tj = S.theta + 7 * (lb + j0 + j);
    double* out = S.theta_next + 7 * (lb + j0 + j);
    for (int a = 0; a < 3; ++a) out[a] = tj[a] + eta * dir[j][a];
    const Q4 qn = normalized(Q4{tj[3] + eta * dir[j][3], tj[4] + eta * dir[j][4], tj[5] + eta * dir[j][5],
                                tj[6] + eta * dir[j][6]});
    out[3] = qn.w;
    out[4] = qn.x;
    out[5] = qn.y;
    out[6] = qn.z;
  }
}

// ---------------------------------------------------------------------------
// K7: SGD update (optim.cpp:108-114) for non-frozen particles.
// ---------------------------------------------------------------------------
__global__ void sgd_kernel(DevProblem P, DevState S) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.J) return;
  double* th = S.theta + 7 * j;
  if (S.converged[j]) return;
  const double* g = S.grad + 7 * j;
  double step[7];
  for (int r = 0; r < 7; ++r) {
    double s = P.A[7 * r] * g[0];
    for (int c = 1; c < 7; ++c) s = s + P.A[7 * r + c] * g[c];
    step[r] = P.lr * s;
  }
  th[0] = th[0] - step[0];
  th[1] = th[1] - step[1];
  th[2] = th[2] - step[2];
  const Q4 qn = normalized(Q4{th[3] - step[3], th[4] - step[4], th[5] - step[5], th[6] - step[6]});
  th[3] = qn.w;
  th[4] = qn.x;
  th[5] = qn.y;
  th[6] = qn.z;
}

// Convergence bookkeeping (grasp.cpp:242-257) and the active mask of the
// next iteration (converged particles freeze in the SGD phase, grasp.cpp:168).
__global__ void bookkeeping_kernel(DevProblem P, DevState S, int stein_phase, int next_stein) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.J) return;
  if (stein_phase) {
    S.prev_loss[j] = S.loss[j];
  } else if (!S.converged[j]) {
    if (S.in_col[j]) {
      S.converged[j] = 0;
    } else {
      const double prev = S.prev_loss[j];
      if (isfinite(prev) && prev > 0.0) S.converged[j] = (fabs(S.loss[j] - prev) / prev <= P.conv_thr) ? 1 : 0;
    }
    S.prev_loss[j] = S.loss[j];
  }
  S.active[j] = (next_stein || !S.converged[j]) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Collision pre-test bounds of one SDF grid, computed at prepare time: the
// Lipschitz bound lip = max |node difference| / voxel along any axis, vmax =
// max |value| (both by atomicMax on the bit patterns of non-negative
// doubles, which order like the values), and the coarse grid: block
// (bx, by, bz) covers cells [4b, 4b + 4) per axis and holds the max over the
// nodes [4b - 1, 4b + 5] (dilated by one node).
// ---------------------------------------------------------------------------
__global__ void grid_bounds_kernel(Grid* grids, int gi, const float* values, float* coarse) {
  Grid& g = grids[gi];
  const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2];
  const float* v = values + g.values_offset;
  const int64_t nodes = static_cast<int64_t>(nx) * ny * nz;
  const int64_t nblocks = static_cast<int64_t>(g.cdims[0]) * g.cdims[1] * g.cdims[2];
  double lip = 0.0, vmax = 0.0;
  for (int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; id < nodes;
       id += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int iz = static_cast<int>(id % nz), iy = static_cast<int>((id / nz) % ny),
              ix = static_cast<int>(id / (static_cast<int64_t>(ny) * nz));
    const double x = v[id];
    vmax = fmax(vmax, fabs(x));
    double d = 0.0;
    if (ix + 1 < nx) d = fmax(d, fabs(x - static_cast<double>(v[id + static_cast<int64_t>(ny) * nz])));
    if (iy + 1 < ny) d = fmax(d, fabs(x - static_cast<double>(v[id + nz])));
    if (iz + 1 < nz) d = fmax(d, fabs(x - static_cast<double>(v[id + 1])));
    lip = fmax(lip, d / g.voxel);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lip = fmax(lip, __shfl_xor_sync(0xffffffffu, lip, o));
    vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(reinterpret_cast<unsigned long long*>(&g.lip), static_cast<unsigned long long>(__double_as_longlong(lip)));
    atomicMax(reinterpret_cast<unsigned long long*>(&g.vmax),
              static_cast<unsigned long long>(__double_as_longlong(vmax)));
  }
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < nblocks;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int bz = static_cast<int>(b % g.cdims[2]), by = static_cast<int>((b / g.cdims[2]) % g.cdims[1]),
              bx = static_cast<int>(b / (static_cast<int64_t>(g.cdims[1]) * g.cdims[2]));
    float m = -INFINITY;
    for (int ix = max(0, kCoarse * bx - 1); ix <= min(nx - 1, kCoarse * bx + kCoarse + 1); ++ix)
      for (int iy = max(0, kCoarse * by - 1); iy <= min(ny - 1, kCoarse * by + kCoarse + 1); ++iy)
        for (int iz = max(0, kCoarse * bz - 1); iz <= min(nz - 1, kCoarse * bz + kCoarse + 1); ++iz)
          m = fmaxf(m, v[(static_cast<int64_t>(ix) * ny + iy) * nz + iz]);
    coarse[g.coarse_offset + b] = m;
  }
}

void launch_grid_bounds(Grid* grids, int n_grids, const float* values, float* coarse, cudaStream_t st) {
  for (int g = 0; g < n_grids; ++g) grid_bounds_kernel<<<296, 256, 0, st>>>(grids, g, values, coarse);
}

// ---------------------------------------------------------------------------
// Particle-sharding exchange: every Stein iteration each
// rank contributes its rows' [theta, drift]; the gathered block is scattered
// into global order so median/svgd read the whole population exactly as the
// unsharded solve does.
// ---------------------------------------------------------------------------
__global__ void pack_stein_kernel(DevProblem P, DevState S, double* send) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.J) return;
  for (int a = 0; a < 7; ++a) {
    send[14 * j + a] = S.theta[7 * j + a];
    send[14 * j + 7 + a] = S.drift[7 * j + a];
  }
}

__global__ void unpack_stein_kernel(const double* gathered, double* theta_all, double* drift_all, int J_glob,
                                    int world, int rows_per_rank) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= world * rows_per_rank) return;
  const int r = row / rows_per_rank, i = row % rows_per_rank;
  const int lo = static_cast<int>(static_cast<int64_t>(r) * J_glob / world);
  const int hi = static_cast<int>(static_cast<int64_t>(r + 1) * J_glob / world);
  if (i >= hi - lo) return;
  const double* src = gathered + 14 * static_cast<int64_t>(row);
  for (int a = 0; a < 7; ++a) {
    theta_all[7 * (lo + i) + a] = src[a];
    drift_all[7 * (lo + i) + a] = src[7 + a];
  }
}

__global__ void pack_final_kernel(DevProblem P, DevState S, double* send, int stride, int k_max, int with_trace) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.J) return;
  double* o = send + static_cast<int64_t>(stride) * j;
  for (int a = 0; a < 7; ++a) o[a] = S.theta[7 * j + a];
  o[7] = S.final_loss[j];
  o[8] = S.final_free[j];
  o[9] = S.converged[j];
  if (!with_trace) return;
  for (int k = 0; k < k_max; ++k) {
    const int64_t r = static_cast<int64_t>(k) * P.J + j;
    double* t = o + 10 + 9 * k;
    for (int a = 0; a < 7; ++a) t[a] = S.trace_theta[7 * r + a];
    t[7] = S.trace_loss[r];
    t[8] = S.trace_col[r];
  }
}

__global__ void copy_theta_kernel(double* dst, const double* src, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

__global__ void init_state_kernel(DevProblem P, DevState S) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.J) return;
  S.loss[j] = __longlong_as_double(0x7ff8000000000000ll);  // quiet NaN (grasp.cpp:124-125)
  S.prev_loss[j] = __longlong_as_double(0x7ff8000000000000ll);
  S.in_col[j] = 0;
  S.converged[j] = 0;
  S.active[j] = 1;
  S.n_col[j] = 0;
}

// FFMA peak probe: 16 independent FFMA chains per thread.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters, float a, float b) {
  float acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = __fmaf_rn(acc[k], a, b);
  }
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  if (s == 1234.5f) out[0] = s;
}

double run_ffma_peak(int iters) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  if (cudaMalloc(&out, 4) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8;
  ffma_peak_kernel<<<blocks, 256>>>(out, iters / 4, 0.999f, 1e-4f);  // warm-up
  cudaEventRecord(e0);
  ffma_peak_kernel<<<blocks, 256>>>(out, iters, 0.999f, 1e-4f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess || ms <= 0.0f) return -1.0;
  const double flops = 2.0 * 16.0 * static_cast<double>(iters) * blocks * 256.0;
  return flops / (ms * 1e-3) / 1e12;
}

__global__ void dbg_exp_kernel(const double* x, double* y, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = glibc_exp(x[i]);
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
void launch_dbg_exp(const double* x, double* y, int64_t n, cudaStream_t st) {
  dbg_exp_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(x, y, n);
}
double host_glibc_exp(double x) { return glibc_exp(x); }

void launch_seed_rng(const DevProblem& P, DevState& S, uint64_t seed, cudaStream_t st) {
  seed_rng_kernel<<<(P.J + 127) / 128, 128, 0, st>>>(S.rng_state, S.rng_mti, seed, P.J);
}
void launch_init_state(const DevProblem& P, DevState& S, cudaStream_t st) {
  init_state_kernel<<<(P.J + 127) / 128, 128, 0, st>>>(P, S);
}
void launch_pose_prep(const DevProblem& P, DevState& S, int all, cudaStream_t st) {
  pose_prep_kernel<<<P.J, kNnThreads, 0, st>>>(P, S, all);
}
void launch_collide(const DevProblem& P, DevState& S, int all, int count_only, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(round_up((P.n_scene + 31) / 32, 4)) * sizeof(unsigned int) +
                      static_cast<size_t>(P.max_coarse) * sizeof(float);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(collide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  collide_kernel<<<P.J, kColThreads, smem, st>>>(P, S, all, count_only);
}
int minibatch_smem_cap() { return 160 * 1024; }

// Opt-in shared-memory sizes of this file's kernels on the current device
// (function attributes are per device: called for every context).
void kernels_set_attrs() {
  cudaFuncSetAttribute(minibatch_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, minibatch_smem_cap());
  cudaFuncSetAttribute(cost_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kCostSmem);
}

void launch_minibatch(const DevProblem& P, DevState& S, int m, cudaStream_t st) {
  if (launch_minibatch_par(P, S, m, st)) return;
  const size_t need = static_cast<size_t>(P.n_obj) * sizeof(int);
  if (need <= static_cast<size_t>(minibatch_smem_cap())) {
    minibatch_kernel<true><<<P.J, 128, need, st>>>(P, S, m);
  } else {
    minibatch_kernel<false><<<P.J, 128, 0, st>>>(P, S, m);
  }
}
void launch_cost(const DevProblem& P, DevState& S, int final_pass, cudaStream_t st) {
  cost_kernel<<<(P.J + 1) / 2, kCostThreads, kCostSmem, st>>>(P, S, final_pass);
}
void launch_trace(const DevProblem& P, DevState& S, int k, cudaStream_t st) {
  trace_kernel<<<(P.J + 127) / 128, 128, 0, st>>>(P, S, k);
}
void launch_drift(const DevProblem& P, DevState& S, double gamma, double n_ref, cudaStream_t st) {
  drift_kernel<<<(P.J + 127) / 128, 128, 0, st>>>(P, S, gamma, n_ref);
}
void launch_pack_stein(const DevProblem& P, const DevState& S, double* send, cudaStream_t st) {
  pack_stein_kernel<<<(P.J + 127) / 128, 128, 0, st>>>(P, S, send);
}
void launch_unpack_stein(const double* gathered, double* theta_all, double* drift_all, int J_glob, int world,
                         int rows_per_rank, cudaStream_t st) {
  const int rows = world * rows_per_rank;
  unpack_stein_kernel<<<(rows + 127) / 128, 128, 0, st>>>(gathered, theta_all, drift_all, J_glob, world,
                                                          rows_per_rank);
}
void launch_pack_final(const DevProblem& P, const DevState& S, double* send, int stride, int k_max, int with_trace,
                       cudaStream_t st) {
  pack_final_kernel<<<(P.J + 127) / 128, 128, 0, st>>>(P, S, send, stride, k_max, with_trace);
}
void launch_svgd_kmat(const DevProblem& P, DevState& S, int max_pop, int max_gpop, cudaStream_t st) {
  svgd_kmat_kernel<<<dim3((max_pop + kSvgdJ - 1) / kSvgdJ, (max_gpop + kSvgdJ - 1) / kSvgdJ, P.n_pop), 256, 0, st>>>(
      P, S);
}

int launch_stein_update(const DevProblem& P, DevState& S, double eta, int max_pop, int max_gpop, int big_grid,
                        cudaStream_t st, bool small_median) {
  int n = 2;
  if (small_median) {
    launch_median_small(P, S, st);
    ++n;
  }
  if (big_grid > 0) {
    med_init_kernel<<<P.n_pop, 256, 0, st>>>(P, S);
    const int shifts[6] = {52, 40, 28, 16, 4, 0}, bits[6] = {12, 12, 12, 12, 12, 4};
    for (int pass = 0; pass < 6; ++pass) {
      med_hist_kernel<<<dim3(big_grid, P.n_pop), 256, 0, st>>>(P, S, shifts[pass], bits[pass]);
      med_select_kernel<<<P.n_pop, 1024, 0, st>>>(P, S, shifts[pass], bits[pass], pass == 5 ? 1 : 0);
    }
    n += 13;
  }
  dim3 grid((max_pop + kSvgdJ - 1) / kSvgdJ, P.n_pop);
  if (S.kmat) {
    // Split SVGD: the kernel matrix needs only the poses and h; with the small
    // median forked (small_median false) the caller launched it on the fork too.
    if (small_median || big_grid > 0) {
      launch_svgd_kmat(P, S, max_pop, max_gpop, st);
      ++n;
    }
    svgd_acc_kernel<<<grid, kSvgdJ * 7, 0, st>>>(P, S, eta);
  } else {
    svgd_kernel<<<grid, kSvgdJ * 7, 0, st>>>(P, S, eta);
  }
  copy_theta_kernel<<<(7 * P.J + 255) / 256, 256, 0, st>>>(S.theta, S.theta_next, 7 * P.J);
  return n;
}
void launch_sgd(const DevProblem& P, DevState& S, cudaStream_t st) {
  sgd_kernel<<<(P.J + 127) / 128, 128, 0, st>>>(P, S);
}
void launch_bookkeeping(const DevProblem& P, DevState& S, int stein_phase, int next_stein, cudaStream_t st) {
  bookkeeping_kernel<<<(P.J + 127) / 128, 128, 0, st>>>(P, S, stein_phase, next_stein);
}

}  // namespace asicp
