// SGD-ICP registration on the device: graspmatch::register_sgd_icp
// (optim.cpp:274-321) with both preconditioners — the fixed matrix
// (sgd_update, optim.cpp:108-114) and the damped Gauss-Newton rotation step
// (gauss_newton_rotation_step, optim.cpp:250-270) — bit-identical to the
// reference (FP64, -fmad=false, the reference's reduction orders).
//
// One CTA per registration problem runs the whole iteration loop: the loop
// is a chain of tiny dependent steps (m = 100 pairs of a 500-point cloud in
// acceptance C2), so a kernel per step would be launch-bound; batching
// independent problems across CTAs is what fills the GPU.  Per iteration:
//   1. the minibatch draw: partial Fisher-Yates over iota(n_source) with
//      std::mt19937_64 + Lemire (spatial_index.cpp:113-125, rng.hpp:32-44),
//      one thread, the array and the 312-word state in shared memory;
//   2. the FP64 nearest neighbour of every transformed batch point in the
//      reference cloud (the kd-tree's "strictly closer, else lowest index",
//      spatial_index.cpp:63-83), brute force: (pair, segment) per thread over
//      the reference staged in shared memory, segments merged in index order;
//   3. per-pair terms (squared distance, residual, the four rotation-gradient
//      dots, the 3x4 Jacobian, its 4x4 moment) written to shared memory in
//      chunks of kRegChunk pairs, then summed left to right by one thread per
//      term — exactly the reference's sequential `+=` over pairs;
//   4. the update on one thread: gradient / m, A g, the Gauss-Newton
//      rotation step (Schur-centred moment, relative damping, the shim's
//      pivot-free LDLT, oracle/shim/Eigen/Dense LdltSolver), pose update,
//      convergence test.
// The rotation_matrix unit-norm require (geometry.cpp:19) is checked every
// iteration; a violation ends the problem with status 1 and the call fails
// with the reference's message.
#include "register.cuh"

#include "common.cuh"
#include "dmath.cuh"
#include "kabsch.cuh"
#include "mt64.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace asicp {
namespace {

constexpr int kRegThreads = 256;
constexpr int kWorkers = 224;      // warps 0-6 match and update; warp 7 draws the next minibatch
constexpr int kRegChunk = 64;      // pairs per accumulation round
constexpr int kTerms = 36;         // |d|^2, residual (3), gradient dots (4), Jacobian (12), moment (16)
constexpr int kTermStride = 37;    // odd stride: conflict-free per-pair rows
constexpr int kPtsSmemMax = 256;   // minibatch points gathered into shared memory (32 B each, double-buffered)
constexpr int kRefSmemMax = 4096;  // FP32 reference candidates staged in shared memory (16 B each)
constexpr int kFySmemMax = 16384;  // Fisher-Yates array in shared memory (4 B each)
constexpr int kBatSmemMax = 2048;  // minibatch double buffer + draws in shared memory (12 B each)
constexpr int kHeadBytes = kRegChunk * kTermStride * 8 + mt::kN * 8;

struct RegCfg {
  double lr, thr, damping;
  double A[49];
  long long max_iter, mb;
  int gn;
};

struct RegArgs {
  const double* src;
  const long long* src_off;
  const double* ref;
  const long long* ref_off;
  const float4* cand;         // FP32 NN candidates (-2b, |b|^2), b = r - centre, one per reference point
  const long long* cand_off;  // per problem: first candidate
  const double* geo;   // per problem: centre (3), B >= max |r - centre|
  const double* init;
  const unsigned long long* seeds;
  int* fy_global;   // per-problem Fisher-Yates arrays for clouds too large for shared memory
  int* bat_global;  // per-problem [2][n_source] minibatches + [n_source] draws (large minibatches)
  double* theta;
  long long* iters;
  double* loss;
  int* conv;
  int* status;
  int ref_cap, fy_cap, bat_cap;  // shared-memory capacities (points / indices / minibatch size)
  int pts_cap;                    // gathered minibatch points per buffer (0: read the source cloud)
  long long pts_off;              // byte offset of the point buffers in dynamic shared memory
  unsigned long long* prof;       // phase clocks of problem 0 (32 words) or null
};

struct alignas(16) P4 {
  double x, y, z, w;
};

__device__ __forceinline__ uint64_t mt_next(uint64_t* s, int* mti) {
  if (*mti >= mt::kN) {
    mt::twist_serial(s);
    *mti = 0;
  }
  return mt::temper(s[(*mti)++]);
}

// Rng::uniform_index (rng.hpp:32-44).
__device__ __forceinline__ uint64_t uniform_index(uint64_t* s, int* mti, uint64_t n) {
  uint64_t out;
  while (!mt::lemire(mt_next(s, mti), n, &out)) {
  }
  return out;
}

// Worker-only barrier (warps 0-6); warp 7 draws the next minibatch meanwhile.
__device__ __forceinline__ void worker_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kWorkers) : "memory"); }

// Warp-cooperative mt19937_64 twist: the in-place recurrence splits into two
// dependency-free halves (mt::twist_block), here with 32 lanes.
__device__ void twist_warp(uint64_t* s, int lane) {
  uint64_t v[5];
  int cnt = 0;
  for (int k = lane; k < mt::kM; k += 32) v[cnt++] = s[k + mt::kM] ^ mt::mix(s[k], s[k + 1]);
  __syncwarp();
  cnt = 0;
  for (int k = lane; k < mt::kM; k += 32) s[k] = v[cnt++];
  __syncwarp();
  cnt = 0;
  for (int k = mt::kM + lane; k < mt::kN; k += 32) v[cnt++] = s[k - mt::kM] ^ mt::mix(s[k], k + 1 < mt::kN ? s[k + 1] : s[0]);
  __syncwarp();
  cnt = 0;
  for (int k = mt::kM + lane; k < mt::kN; k += 32) s[k] = v[cnt++];
  __syncwarp();
}

// sample_minibatch_indices (spatial_index.cpp:113-125) by one warp: the m
// Lemire draws (rng.hpp:32-44) are reduced 32 at a time from consecutive
// engine outputs; a rejected output (lo < (2^64 - n) mod n) is consumed and
// its draw retried with the next output, exactly like the serial loop.  The
// swaps of the partial Fisher-Yates then run on lane 0 (bat[i] = idx[i]
// after swap i).  The engine twists lazily, when an output is needed.
__device__ void draw_batch(uint64_t* mts, int& mti, int* fy, int* jv, int* bat, int n_src, int m, int lane) {
  for (int i = lane; i < n_src; i += 32) fy[i] = i;
  int i0 = 0;
  while (i0 < m) {
    if (mti >= mt::kN) {
      twist_warp(mts, lane);
      mti = 0;
    }
    const int take = min(min(32, m - i0), mt::kN - mti);
    bool ok = true;
    uint64_t j = 0;
    if (lane < take) ok = mt::lemire(mt::temper(mts[mti + lane]), static_cast<uint64_t>(n_src - (i0 + lane)), &j);
    const unsigned rej = __ballot_sync(0xffffffffu, !ok);
    const int valid = rej ? __ffs(rej) - 1 : take;
    if (lane < valid) jv[i0 + lane] = i0 + lane + static_cast<int>(j);
    mti += rej ? valid + 1 : take;
    i0 += valid;
  }
  __syncwarp();
  if (lane == 0)
    for (int i = 0; i < m; ++i) {
      const int j = jv[i];
      const int v = fy[j];
      fy[j] = fy[i];
      bat[i] = v;
    }
}

// Thread 0, after the parallel phase: the serial tail of
// gauss_newton_rotation_step (optim.cpp:265-269) — trace, relative damping,
// the shim's pivot-free LDLT solve (oracle/shim/Eigen/Dense LdltSolver).
__device__ void gn_solve(const double* cen, const double* gc, const double* g, double damping, double* dq) {
  const double trace = ((cen[0] + cen[5]) + cen[10]) + cen[15];
  if (!(trace > 1e-12)) {
    for (int i = 0; i < 4; ++i) dq[i] = g[3 + i];
    return;
  }
  const double sd = damping * trace / 4.0;
  double l[4][4] = {{1.0, 0.0, 0.0, 0.0}, {0.0, 1.0, 0.0, 0.0}, {0.0, 0.0, 1.0, 0.0}, {0.0, 0.0, 0.0, 1.0}};
  double dv[4];
  for (int j = 0; j < 4; ++j) {
    double s = cen[5 * j] + sd * 1.0;
    for (int k = 0; k < j; ++k) s = s - l[j][k] * l[j][k] * dv[k];
    dv[j] = s;
    for (int i = j + 1; i < 4; ++i) {
      double t = cen[4 * i + j] + sd * 0.0;
      for (int k = 0; k < j; ++k) t = t - l[i][k] * l[j][k] * dv[k];
      l[i][j] = t / dv[j];
    }
  }
  double y[4];
  for (int i = 0; i < 4; ++i) {
    double s = gc[i];
    for (int k = 0; k < i; ++k) s = s - l[i][k] * y[k];
    y[i] = s;
  }
  for (int i = 0; i < 4; ++i) y[i] = y[i] / dv[i];
  for (int i = 3; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 4; ++k) s = s - l[k][i] * dq[k];
    dq[i] = s;
  }
}

// Thread 0: the rotation_matrix require for the pose of the next iteration
// (geometry.cpp:19), then R and dR/dq into shared memory.  False = violated.
__device__ bool pose_setup(const double* th, double* s_R, double* s_dR) {
  const Q4 q{th[3], th[4], th[5], th[6]};
  if (!(fabs(sqrt(sqnorm4(q)) - 1.0) <= 1e-6)) return false;
  const M3 R = rotation_matrix(q);
  M3 d[4];
  rotation_matrix_derivatives(q, d);
  for (int i = 0; i < 9; ++i) {
    s_R[i] = R.m[i];
    for (int j = 0; j < 4; ++j) s_dR[9 * j + i] = d[j].m[i];
  }
  return true;
}

// One query against candidates [lo, hi) in one FP32 pass that keeps the
// smallest d32 (b1, at i1) and the second smallest (b2).  The window
// {d32 <= b1 + 2E} holds the exact FP64 answer; when b2 is outside it, i1 is
// its only member and one FP64 distance settles the query (uniform across
// the warp).  Otherwise the members are evaluated in FP64 in index order,
// strictly closer wins (the kd-tree's rule).  Candidates here are stored one
// float4 per point (cand1).
__device__ __forceinline__ void nn_window(const float4* cnd, const double* refg, int lo, int hi, const V3& q,
                                          float qx, float qy, float qz, float mg, double& best, int& bi) {
  float b1 = INFINITY, b2 = INFINITY;
  int i1 = -1;
#pragma unroll 8
  for (int i = lo; i < hi; ++i) {
    const float4 v = cnd[i];
    const float d = __fmaf_rn(qx, v.x, __fmaf_rn(qy, v.y, __fmaf_rn(qz, v.z, v.w)));
    b2 = fminf(b2, fmaxf(b1, d));
    i1 = d < b1 ? i : i1;
    b1 = fminf(b1, d);
  }
  if (i1 < 0) return;  // empty segment
  const float lim = __fadd_ru(b1, mg);
  if (b2 > lim) {
    best = sqnorm(sub(load3(refg, i1), q));
    bi = i1;
    return;
  }
  for (int i = lo; i < hi; ++i) {
    const float4 v = cnd[i];
    if (__fmaf_rn(qx, v.x, __fmaf_rn(qy, v.y, __fmaf_rn(qz, v.z, v.w))) <= lim) {
      const double d2 = sqnorm(sub(load3(refg, i), q));
      if (d2 < best) {
        best = d2;
        bi = i;
      }
    }
  }
}

__global__ void __launch_bounds__(kRegThreads, 4) register_kernel(RegArgs a, RegCfg c) {
  const int p = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  extern __shared__ __align__(16) unsigned char reg_smem[];
  double* terms = reinterpret_cast<double*>(reg_smem);
  uint64_t* mts = reinterpret_cast<uint64_t*>(terms + kRegChunk * kTermStride);
  float4* cands = reinterpret_cast<float4*>(mts + mt::kN);
  int* fy_smem = reinterpret_cast<int*>(cands + a.ref_cap);
  int* bat_smem = fy_smem + a.fy_cap;  // [2][bat_cap] minibatches + [bat_cap] draws
  P4* pts = reinterpret_cast<P4*>(reg_smem + a.pts_off);  // [2][pts_cap] gathered minibatch points
  __shared__ double s_th[7], s_R[9], s_dR[36], s_div[kTerms], s_pre[7], s_cen[16], s_gc[4];
  __shared__ double s_nnd[kWorkers];
  __shared__ int s_nni[kWorkers];
  __shared__ P4 s_q64[kRegChunk];      // chunk queries, FP64 (transformed minibatch points)
  __shared__ int s_stop, s_status;

  const long long s0 = a.src_off[p], r0 = a.ref_off[p];
  const int n_src = static_cast<int>(a.src_off[p + 1] - s0), n_ref = static_cast<int>(a.ref_off[p + 1] - r0);
  const double* src = a.src + 3 * s0;
  const double* refg = a.ref + 3 * r0;
  const bool ref_in = n_ref <= a.ref_cap;
  const int m = static_cast<int>(c.mb < n_src ? c.mb : n_src);
  int* fy = n_src <= a.fy_cap ? fy_smem : a.fy_global + s0;
  int* bat = m <= a.bat_cap ? bat_smem : a.bat_global + 3 * s0;
  const int bat_stride = m <= a.bat_cap ? a.bat_cap : n_src;
  int* jv = bat + 2 * bat_stride;
  const int nterms = c.gn ? kTerms : 8;
  const bool pts_in = m <= a.pts_cap;

  const float4* candg = a.cand + a.cand_off[p];
  if (ref_in)
    for (int i = tid; i < n_ref; i += kRegThreads) cands[i] = candg[i];
  const double cx = a.geo[4 * p], cy = a.geo[4 * p + 1], cz = a.geo[4 * p + 2], Bp = a.geo[4 * p + 3];
  int mti = mt::kN, conv = 0, status = 0;
  long long iters = 0;
  double prev_loss = -1.0, final_loss = 0.0;
  // Phase clock (diagnostics; build with -DASICP_REG_PHASES and set
  // ASICP_REG_PROFILE=1): problem 0's worker thread 0 and drawer lane 0
  // accumulate clock64 deltas per phase.
#ifdef ASICP_REG_PHASES
  const bool prof_on = a.prof != nullptr && p == 0 && (tid == 0 || tid == kWorkers);
  unsigned long long ph[14] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_last = clock64();
#define PH(i)                                  \
  do {                                         \
    if (prof_on) {                             \
      const long long now_ = clock64();        \
      ph[i] += now_ - ph_last;                 \
      ph_last = now_;                          \
    }                                          \
  } while (0)
#else
#define PH(i) \
  do {        \
  } while (0)
#endif
  if (tid == 0) {
    s_stop = 0;
    s_status = 0;
    for (int i = 0; i < 7; ++i) s_th[i] = a.init[7 * static_cast<long long>(p) + i];
    if (c.max_iter > 0 && !pose_setup(s_th, s_R, s_dR)) {
      status = 1;
      s_stop = 1;
    }
  }
  if (warp == kWorkers / 32) {
    if (lane == 0) mt::seed_state(mts, a.seeds[p]);
    __syncwarp();
    if (c.max_iter > 0) {
      draw_batch(mts, mti, fy, jv, bat, n_src, m, lane);
      __syncwarp();
      if (pts_in)
        for (int i = lane; i < m; i += 32) {
          const V3 v = load3(src, bat[i]);
          pts[i] = P4{v.x, v.y, v.z, 0.0};
        }
    }
  }
  __syncthreads();

  for (long long k = 0; k < c.max_iter && !s_stop; ++k) {
    PH(0);
    if (warp == kWorkers / 32) {
      PH(8);
      if (k + 1 < c.max_iter) {
        const int nb = (k + 1) & 1;
        draw_batch(mts, mti, fy, jv, bat + nb * bat_stride, n_src, m, lane);
        __syncwarp();
        if (pts_in)  // gather the next minibatch's source points
          for (int i = lane; i < m; i += 32) {
            const V3 v = load3(src, bat[nb * bat_stride + i]);
            pts[nb * a.pts_cap + i] = P4{v.x, v.y, v.z, 0.0};
          }
      }
      PH(9);
    } else {
      const int* cur = bat + (k & 1) * bat_stride;
      const P4* cpts = pts + (k & 1) * a.pts_cap;
      M3 R;
      for (int i = 0; i < 9; ++i) R.m[i] = s_R[i];
      const V3 t{s_th[0], s_th[1], s_th[2]};
      auto point = [&](int i) {  // minibatch point i (source frame)
        if (pts_in) {
          const P4 v = cpts[i];
          return V3{v.x, v.y, v.z};
        }
        return load3(src, cur[i]);
      };
      double acc = 0.0;
      for (int c0 = 0; c0 < m; c0 += kRegChunk) {
        const int np = m - c0 < kRegChunk ? m - c0 : kRegChunk;
        // (A) thread = (query, candidate segment): certified FP32 filter,
        // FP64 distance of the window member(s).
        const int nseg = kWorkers / np;  // >= 3
        if (tid < np * nseg) {
          const int qi = tid % np, seg = tid / np;
          const V3 q = transform(R, t, point(c0 + qi));
          const int lo = static_cast<int>(static_cast<long long>(n_ref) * seg / nseg);
          const int hi = static_cast<int>(static_cast<long long>(n_ref) * (seg + 1) / nseg);
          const double ax = q.x - cx, ay = q.y - cy, az = q.z - cz;
          const double A = sqrt(ax * ax + ay * ay + az * az);
          double best = INFINITY;
          int bi = -1;
          if (!(A < 1e15 && Bp < 1e15)) {
            for (int i = lo; i < hi; ++i) {  // far outside FP32's range: plain FP64 scan
              const double d2 = sqnorm(sub(load3(refg, i), q));
              if (d2 < best) {
                best = d2;
                bi = i;
              }
            }
          } else {
            const float fx = __double2float_rn(ax), fy = __double2float_rn(ay), fz = __double2float_rn(az);
            if (ref_in)
              nn_window(cands, refg, lo, hi, q, fx, fy, fz, nn_margin(A, Bp), best, bi);
            else
              nn_window(candg, refg, lo, hi, q, fx, fy, fz, nn_margin(A, Bp), best, bi);
          }
          s_nnd[tid] = best;
          s_nni[tid] = bi;
          if (seg == 0) s_q64[qi] = P4{q.x, q.y, q.z, 0.0};
        }
        worker_sync();
        PH(1);
        // (B) thread = pair: the segments hold increasing index ranges, so an
        // equal distance keeps the earlier (lower-index) answer; then every
        // per-pair term of the sums.
        if (tid < np) {
          double best = s_nnd[tid];
          int bi = s_nni[tid];
          for (int sg = 1; sg < nseg; ++sg)
            if (s_nnd[sg * np + tid] < best) {
              best = s_nnd[sg * np + tid];
              bi = s_nni[sg * np + tid];
            }
          const P4 q4 = s_q64[tid];
          const V3 q{q4.x, q4.y, q4.z};
          if (bi < 0) bi = 0;  // unreachable for finite clouds
          PH(11);
          const V3 s = point(c0 + tid);
          const V3 rp = load3(refg, bi);
          double* tm = terms + tid * kTermStride;
          const double dist = sqrt(best);
          tm[0] = dist * dist;
          const V3 res = sub(q, rp);
          tm[1] = res.x;
          tm[2] = res.y;
          tm[3] = res.z;
          V3 v[4];
          for (int j = 0; j < 4; ++j) {
            M3 dj;
            for (int i = 0; i < 9; ++i) dj.m[i] = s_dR[9 * j + i];
            v[j] = mul(dj, s);
            tm[4 + j] = dot(res, v[j]);
          }
          if (c.gn) {
            for (int j = 0; j < 4; ++j) {
              tm[8 + 3 * j] = v[j].x;
              tm[9 + 3 * j] = v[j].y;
              tm[10 + 3 * j] = v[j].z;
            }
            for (int i = 0; i < 4; ++i)  // (jac^T jac)(i, j), optim.cpp:261
              for (int j = 0; j < 4; ++j) tm[20 + 4 * i + j] = dot(v[i], v[j]);
          }
          PH(12);
        }
        worker_sync();
        PH(2);
        // (C) The reference's sequential `+=` over pairs, one thread per sum;
        // operands are loaded 8 steps ahead so only the additions chain.
        if (tid < nterms) {
          int i = 0;
          for (; i + 8 <= np; i += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = terms[(i + u) * kTermStride + tid];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = acc + v[u];
          }
          for (; i < np; ++i) acc = acc + terms[i * kTermStride + tid];
        }
        worker_sync();
        PH(3);
      }
      // Every mean at once: loss, g (optim.cpp:103-104), jac_mean and moment
      // (optim.cpp:262-263) are each a sum / m.
      const double md = static_cast<double>(m);
      if (tid < nterms) s_div[tid] = acc / md;
      worker_sync();
      PH(4);
      const double* g = s_div + 1;
      if (tid < 7) {  // A g (optim.cpp:109 / 303)
        double s2 = c.A[7 * tid] * g[0];
        for (int k2 = 1; k2 < 7; ++k2) s2 = s2 + c.A[7 * tid + k2] * g[k2];
        s_pre[tid] = s2;
      } else if (c.gn && tid >= 32 && tid < 48) {  // centered = moment - jac_mean^T jac_mean
        const int i = (tid - 32) >> 2, j = (tid - 32) & 3;
        const double* jm = s_div + 8;  // jm(r, j) = jm[3 j + r]
        s_cen[tid - 32] = s_div[20 + 4 * i + j] -
                          ((jm[3 * i] * jm[3 * j] + jm[3 * i + 1] * jm[3 * j + 1]) + jm[3 * i + 2] * jm[3 * j + 2]);
      } else if (c.gn && tid >= 64 && tid < 68) {  // g_centered = g_q - jac_mean^T g_t
        const int i = tid - 64;
        const double* jm = s_div + 8;
        s_gc[i] = g[3 + i] - ((jm[3 * i] * g[0] + jm[3 * i + 1] * g[1]) + jm[3 * i + 2] * g[2]);
      }
      worker_sync();
      PH(5);
      if (tid == 0) {
        const double loss = s_div[0];
        double dq[4];
        if (!c.gn) {
          for (int i = 0; i < 4; ++i) dq[i] = s_pre[3 + i];  // sgd_update: q - lr (A g).tail
        } else {
          gn_solve(s_cen, s_gc, g, c.damping, dq);
        }
        for (int i = 0; i < 3; ++i) s_th[i] = s_th[i] - c.lr * s_pre[i];
        const Q4 qn = normalized(
            Q4{s_th[3] - c.lr * dq[0], s_th[4] - c.lr * dq[1], s_th[5] - c.lr * dq[2], s_th[6] - c.lr * dq[3]});
        s_th[3] = qn.w;
        s_th[4] = qn.x;
        s_th[5] = qn.y;
        s_th[6] = qn.z;
        iters = k + 1;
        final_loss = loss;
        if (prev_loss > 0.0 && c.thr >= 0.0 && fabs(loss - prev_loss) / prev_loss <= c.thr && m == n_src) {
          conv = 1;
          s_stop = 1;
        }
        prev_loss = loss;
      }
      worker_sync();
      // Next pose's rotation (geometry.cpp:8-32) in parallel, and the
      // rotation_matrix unit-norm require of the next iteration (:19).
      if (!s_stop && k + 1 < c.max_iter) {
        const Q4 q{s_th[3], s_th[4], s_th[5], s_th[6]};
        if (tid < 9) {  // R = homogeneous / |q|^2, one entry per thread
          const M3 h = rotation_matrix_homogeneous(q);
          double v = 0.0;
#pragma unroll
          for (int i = 0; i < 9; ++i)
            if (i == tid) v = h.m[i];
          s_R[tid] = v / sqnorm4(q);
        } else if (tid == 32) {
          M3 d[4];
          rotation_matrix_derivatives(q, d);
          for (int j = 0; j < 4; ++j)
            for (int i = 0; i < 9; ++i) s_dR[9 * j + i] = d[j].m[i];
        } else if (tid == 64) {
          if (!(fabs(sqrt(sqnorm4(q)) - 1.0) <= 1e-6)) {
            s_status = 1;
            s_stop = 1;
          }
        }
      }
      PH(6);
    }
    __syncthreads();
    PH(7);
  }
  if (tid == 0 && s_status) status = 1;
#ifdef ASICP_REG_PHASES
  if (prof_on) {
    unsigned long long* out = a.prof + (tid == 0 ? 0 : 16);  // 15 words each
    for (int i = 0; i < 14; ++i) out[i] = ph[i];
    out[14] = iters;
  }
#endif
  if (tid == 0) {
    for (int i = 0; i < 7; ++i) a.theta[7 * static_cast<long long>(p) + i] = s_th[i];
    a.iters[p] = iters;
    a.loss[p] = final_loss;
    a.conv[p] = conv;
    a.status[p] = status;
  }
}

// FP32 NN candidates of every problem's reference cloud, one CTA per problem:
// centre c = the cloud's mean (any fixed point works — the certification
// bound B is measured from the same c), b = r - c rounded to FP32,
// (-2b, |b|^2) as the forward match builds them (solver.cu prepare), and
// B = max |r - c| with slack.
__global__ void __launch_bounds__(256) reg_cand_kernel(const double* ref, const long long* ref_off, float4* cand,
                                                       double* geo) {
  const int p = blockIdx.x, tid = threadIdx.x;
  const long long r0 = ref_off[p];
  const int nr = static_cast<int>(ref_off[p + 1] - r0);
  const double* r = ref + 3 * r0;
  __shared__ double red[3][256];
  __shared__ double s_c[3];
  double sx = 0.0, sy = 0.0, sz = 0.0;
  for (int i = tid; i < nr; i += 256) {
    sx += r[3 * i];
    sy += r[3 * i + 1];
    sz += r[3 * i + 2];
  }
  red[0][tid] = sx;
  red[1][tid] = sy;
  red[2][tid] = sz;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (tid < off)
      for (int a = 0; a < 3; ++a) red[a][tid] += red[a][tid + off];
    __syncthreads();
  }
  if (tid < 3) s_c[tid] = red[tid][0] / static_cast<double>(nr);
  __syncthreads();
  const double cx = s_c[0], cy = s_c[1], cz = s_c[2];
  double bmax = 0.0;
  for (int i = tid; i < nr; i += 256) {
    const double bx = r[3 * i] - cx, by = r[3 * i + 1] - cy, bz = r[3 * i + 2] - cz;
    const float fx = __double2float_rn(bx), fy = __double2float_rn(by), fz = __double2float_rn(bz);
    const double dx = fx, dy = fy, dz = fz;
    cand[r0 + i] = make_float4(-2.0f * fx, -2.0f * fy, -2.0f * fz, __double2float_rn(dx * dx + dy * dy + dz * dz));
    bmax = fmax(bmax, sqrt(bx * bx + by * by + bz * bz));
  }
  __syncthreads();
  red[0][tid] = bmax;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (tid < off) red[0][tid] = fmax(red[0][tid], red[0][tid + off]);
    __syncthreads();
  }
  if (tid == 0) {
    geo[4 * p] = cx;
    geo[4 * p + 1] = cy;
    geo[4 * p + 2] = cz;
    geo[4 * p + 3] = red[0][0] * (1.0 + 1e-6) + 1e-12;
  }
}

// graspmatch::icp_closed_form_step (optim.cpp:51-90), one CTA per problem:
// every source point transformed by theta and matched in the reference (the
// certified FP32 filter + FP64 check of the registration kernel), the means
// and the covariance as the reference's sequential sums (one thread each, in
// source order), then the SVD / Kabsch / quaternion tail on thread 0.
struct IcpArgs {
  const double* src;
  const long long* src_off;
  const double* ref;
  const long long* ref_off;
  const float4* cand;
  const double* geo;
  const double* theta;  // n x 7 input poses
  int* match;           // per source point: matched reference index
  double* out;          // n x 7
  int* degenerate;
};

__global__ void __launch_bounds__(256) icp_step_kernel(IcpArgs a) {
  const int p = blockIdx.x, tid = threadIdx.x;
  const long long s0 = a.src_off[p], r0 = a.ref_off[p];
  const int n_src = static_cast<int>(a.src_off[p + 1] - s0), n_ref = static_cast<int>(a.ref_off[p + 1] - r0);
  const double* src = a.src + 3 * s0;
  const double* refg = a.ref + 3 * r0;
  const float4* candg = a.cand + r0;
  int* match = a.match + s0;
  const double* th = a.theta + 7 * static_cast<long long>(p);
  const double cx = a.geo[4 * p], cy = a.geo[4 * p + 1], cz = a.geo[4 * p + 2], Bp = a.geo[4 * p + 3];
  __shared__ double s_mean[6], s_cov[9];
  const M3 R = rotation_matrix(pose_q(th));  // apply_transform (geometry.cpp:68-74); unit norm checked on the host
  const V3 t = pose_t(th);
  for (int i = tid; i < n_src; i += blockDim.x) {
    const V3 q = transform(R, t, load3(src, i));
    const double ax = q.x - cx, ay = q.y - cy, az = q.z - cz;
    const double A = sqrt(ax * ax + ay * ay + az * az);
    double best = INFINITY;
    int bi = -1;
    if (!(A < 1e15 && Bp < 1e15)) {
      for (int k = 0; k < n_ref; ++k) {
        const double d2 = sqnorm(sub(load3(refg, k), q));
        if (d2 < best) {
          best = d2;
          bi = k;
        }
      }
    } else {
      nn_window(candg, refg, 0, n_ref, q, __double2float_rn(ax), __double2float_rn(ay), __double2float_rn(az),
                nn_margin(A, Bp), best, bi);
    }
    match[i] = bi < 0 ? 0 : bi;
  }
  __syncthreads();
  const double nd = static_cast<double>(n_src);
  if (tid < 6) {  // ref_mean += match; src_mean += s (optim.cpp:57-62)
    double acc = 0.0;
    if (tid < 3)
      for (int i = 0; i < n_src; ++i) acc = acc + refg[3 * match[i] + tid];
    else
      for (int i = 0; i < n_src; ++i) acc = acc + src[3 * i + tid - 3];
    s_mean[tid] = acc / nd;
  }
  __syncthreads();
  if (tid < 9) {  // cov += (s - src_mean)(match - ref_mean)^T (optim.cpp:64-66)
    const int r = tid / 3, c = tid % 3;
    const double sm = s_mean[3 + r], rm = s_mean[c];
    double acc = 0.0;
    for (int i = 0; i < n_src; ++i) acc = acc + (src[3 * i + r] - sm) * (refg[3 * match[i] + c] - rm);
    s_cov[tid] = acc;
  }
  __syncthreads();
  if (tid == 0) {
    Mat3 cov;
    for (int i = 0; i < 9; ++i) cov.a[i / 3][i % 3] = s_cov[i];
    a.degenerate[p] = kabsch_finish(th, V3{s_mean[3], s_mean[4], s_mean[5]}, V3{s_mean[0], s_mean[1], s_mean[2]}, cov,
                                    n_src, a.out + 7 * static_cast<long long>(p));
  }
}

// Host restatements of SgdConfig::validate (optim.cpp:10-15) against the
// shim's isApprox / LLT (oracle/shim/Eigen/Dense).
double col_major_norm(const double* A, bool transposed) {
  auto at = [&](int i, int j) { return transposed ? A[7 * j + i] : A[7 * i + j]; };
  double s = at(0, 0) * at(0, 0);
  for (int j = 0; j < 7; ++j)
    for (int i = 0; i < 7; ++i)
      if (i != 0 || j != 0) s = s + at(i, j) * at(i, j);
  return std::sqrt(s);
}

bool sgd_symmetric(const double* A) {
  double d[49];
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) d[7 * i + j] = A[7 * i + j] - A[7 * j + i];
  return col_major_norm(d, false) <= 1e-12 * std::min(col_major_norm(A, false), col_major_norm(A, true));
}

bool sgd_llt_ok(const double* A) {
  double l[7][7];
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) l[i][j] = A[7 * i + j];
  for (int j = 0; j < 7; ++j) {
    double s = l[j][j];
    for (int k = 0; k < j; ++k) s -= l[j][k] * l[j][k];
    if (!(s > 0.0)) return false;
    const double dd = std::sqrt(s);
    l[j][j] = dd;
    for (int i = j + 1; i < 7; ++i) {
      double t = l[i][j];
      for (int k = 0; k < j; ++k) t -= l[i][k] * l[j][k];
      l[i][j] = t / dd;
    }
    for (int i = 0; i < j; ++i) l[i][j] = 0.0;
  }
  return true;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

}  // namespace

// FP64 throughput ceiling of this GPU (DFMA, 2 FLOP each): the roofline
// denominator of the registration kernel's brute-force NN, which cannot
// contract (bit-exactness) and so tops out at half of it.
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = __fma_rn(acc[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  if (s == 1234.5) out[0] = s;
}

struct RegBatch::Dev {
  int n = 0;
  RegCfg cfg{};
  int ref_cap = 0, fy_cap = 0, bat_cap = 0, pts_cap = 0;
  long long pts_off = 0;
  size_t smem = 0;
  DevBuf src, src_off, ref, ref_off, cand, cand_off, geo, init, seeds, fy, bat, theta, iters, loss, conv, status, prof;
  // Pinned result staging.
  double* h_theta = nullptr;
  long long* h_iters = nullptr;
  double* h_loss = nullptr;
  int* h_conv = nullptr;
  int* h_status = nullptr;
  int h_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void free_host() {
    void* all[] = {h_theta, h_iters, h_loss, h_conv, h_status};
    for (void* q : all)
      if (q) cudaFreeHost(q);
    h_theta = nullptr;
    h_iters = nullptr;
    h_loss = nullptr;
    h_conv = nullptr;
    h_status = nullptr;
    h_cap = 0;
  }
  ~Dev() {
    free_host();
    DevBuf* all[] = {&src, &src_off, &ref,  &ref_off, &cand, &cand_off, &geo,  &init,  &seeds,
                     &fy,  &bat,     &theta, &iters,   &loss, &conv, &status, &prof};
    for (DevBuf* b : all) b->release();
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
  }
};

RegBatch::~RegBatch() { release(); }

void RegBatch::release() {
  delete d_;
  d_ = nullptr;
  delete icp_;
  icp_ = nullptr;
}

#define REG_CUDA(expr)                                                                    \
  do {                                                                                    \
    const cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) {                                                              \
      *err = std::string(#expr) + ": " + cudaGetErrorString(e_);                          \
      return ASICP_DEVICE_ERROR;                                                          \
    }                                                                                     \
  } while (0)

int RegBatch::prepare(int64_t n, const double* sources, const int64_t* src_off, const double* references,
                      const int64_t* ref_off, const double* initial, const uint64_t* seeds,
                      const asicp_sgd_config& cfg, std::string* err) {
  auto invalid = [&](const char* msg) {
    *err = msg;
    return ASICP_INVALID_ARGUMENT;
  };
  if (n < 0) return invalid("asicp: negative problem count");
  if (cfg.max_iterations < 0 || cfg.minibatch_size < 0)
    return invalid("asicp: max_iterations and minibatch_size must be >= 0");
  if (cfg.preconditioner_mode != ASICP_PRECOND_FIXED && cfg.preconditioner_mode != ASICP_PRECOND_GAUSS_NEWTON_ROTATION)
    return invalid("asicp: unknown preconditioner_mode");
  if (n > (1ll << 31) - 1) return invalid("asicp: too many problems");
  if (n > 0 && (!src_off || !ref_off || !initial || !seeds)) return invalid("asicp: null batch array");
  int max_src = 0, max_ref = 0, max_m = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t ns = src_off[i + 1] - src_off[i], nr = ref_off[i + 1] - ref_off[i];
    // register_sgd_icp (optim.cpp:277-290), in the reference's order.
    if (ns < 0 || nr < 0) return invalid("asicp: decreasing cloud offsets");
    if (ns == 0 || nr == 0) return invalid("register_sgd_icp: empty cloud");
    if (cfg.preconditioner_mode == ASICP_PRECOND_FIXED) {
      if (!(cfg.learning_rate > 0.0)) return invalid("SgdConfig: learning_rate must be positive");
      if (!sgd_symmetric(cfg.A)) return invalid("SgdConfig: A must be symmetric");
      if (!sgd_llt_ok(cfg.A)) return invalid("SgdConfig: A must be positive definite");
    }
    if (ns >= (1ll << 31) || nr >= (1ll << 31)) return invalid("asicp: cloud too large");
    if (cfg.max_iterations > 0) {
      if (std::min<int64_t>(cfg.minibatch_size, ns) < 1) return invalid("sample_minibatch: m out of range");
      const double* q = initial + 7 * i + 3;
      const double n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
      if (!(std::abs(std::sqrt(n2) - 1.0) <= 1e-6)) return invalid("rotation_matrix: quaternion is not unit-norm");
    }
    max_src = std::max<int>(max_src, static_cast<int>(ns));
    max_m = std::max<int>(max_m, static_cast<int>(std::min<int64_t>(cfg.minibatch_size, ns)));
    max_ref = std::max<int>(max_ref, static_cast<int>(nr));
  }
  REG_CUDA(cudaSetDevice(device_));
  if (!d_) d_ = new Dev();
  Dev& D = *d_;
  D.n = static_cast<int>(n);
  D.cfg.lr = cfg.learning_rate;
  D.cfg.thr = cfg.convergence_threshold;
  D.cfg.damping = cfg.gn_damping;
  std::memcpy(D.cfg.A, cfg.A, sizeof(D.cfg.A));
  D.cfg.max_iter = cfg.max_iterations;
  D.cfg.mb = cfg.minibatch_size;
  D.cfg.gn = cfg.preconditioner_mode == ASICP_PRECOND_GAUSS_NEWTON_ROTATION ? 1 : 0;
  D.ref_cap = max_ref <= kRefSmemMax ? max_ref : 0;
  D.fy_cap = max_src <= kFySmemMax ? max_src : 0;
  D.bat_cap = max_m <= kBatSmemMax ? max_m : 0;
  D.pts_cap = max_m <= kPtsSmemMax ? max_m : 0;
  D.smem = kHeadBytes + static_cast<size_t>(D.ref_cap) * sizeof(float4) +
           static_cast<size_t>(D.fy_cap) * 4 + static_cast<size_t>(D.bat_cap) * 12;
  D.smem = (D.smem + 15) / 16 * 16;
  D.pts_off = static_cast<long long>(D.smem);
  D.smem += static_cast<size_t>(D.pts_cap) * 2 * sizeof(P4);
  if (n == 0) return ASICP_OK;
  const int64_t tot_src = src_off[n] - src_off[0], tot_ref = ref_off[n] - ref_off[0];
  // Offsets are rebased to the first problem's rows.
  std::vector<long long> so(n + 1), ro(n + 1);
  for (int64_t i = 0; i <= n; ++i) {
    so[i] = src_off[i] - src_off[0];
    ro[i] = ref_off[i] - ref_off[0];
  }
  REG_CUDA(D.src.ensure(std::max<int64_t>(tot_src, 1) * 24));
  REG_CUDA(D.ref.ensure(std::max<int64_t>(tot_ref, 1) * 24));
  REG_CUDA(D.src_off.ensure((n + 1) * 8));
  REG_CUDA(D.ref_off.ensure((n + 1) * 8));
  REG_CUDA(D.init.ensure(n * 56));
  REG_CUDA(D.seeds.ensure(n * 8));
  REG_CUDA(D.fy.ensure(D.fy_cap ? 4 : std::max<int64_t>(tot_src, 1) * 4));
  REG_CUDA(D.bat.ensure(D.bat_cap ? 4 : std::max<int64_t>(tot_src, 1) * 12));
  REG_CUDA(D.theta.ensure(n * 56));
  REG_CUDA(D.iters.ensure(n * 8));
  REG_CUDA(D.loss.ensure(n * 8));
  REG_CUDA(D.conv.ensure(n * 4));
  REG_CUDA(D.status.ensure(n * 4));
  REG_CUDA(cudaMemcpyAsync(D.src.p, sources + 3 * src_off[0], tot_src * 24, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.ref.p, references + 3 * ref_off[0], tot_ref * 24, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.src_off.p, so.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.ref_off.p, ro.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st_));
  REG_CUDA(D.cand.ensure(static_cast<size_t>(std::max<int64_t>(tot_ref, 1)) * sizeof(float4)));
  REG_CUDA(D.geo.ensure(static_cast<size_t>(n) * 4 * 8));
  reg_cand_kernel<<<static_cast<unsigned>(n), 256, 0, st_>>>(static_cast<const double*>(D.ref.p),
                                                             static_cast<const long long*>(D.ref_off.p),
                                                             static_cast<float4*>(D.cand.p),
                                                             static_cast<double*>(D.geo.p));
  REG_CUDA(cudaGetLastError());
  REG_CUDA(cudaMemcpyAsync(D.init.p, initial, n * 56, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.seeds.p, seeds, n * 8, cudaMemcpyHostToDevice, st_));
  if (D.h_cap < n) {
    D.free_host();
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_theta), n * 56));
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_iters), n * 8));
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_loss), n * 8));
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_conv), n * 4));
    REG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&D.h_status), n * 4));
    D.h_cap = static_cast<int>(n);
  }
  if (!D.ev0) REG_CUDA(cudaEventCreate(&D.ev0));
  if (!D.ev1) REG_CUDA(cudaEventCreate(&D.ev1));
  REG_CUDA(cudaFuncSetAttribute(register_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(D.smem)));
  // The upload reads caller memory: finish it before returning.
  REG_CUDA(cudaStreamSynchronize(st_));
  return ASICP_OK;
}

int RegBatch::icp_step(int64_t n, const double* sources, const int64_t* src_off, const double* references,
                       const int64_t* ref_off, const double* thetas, asicp_icp_step* out, std::string* err) {
  auto invalid = [&](const char* msg) {
    *err = msg;
    return ASICP_INVALID_ARGUMENT;
  };
  if (n < 0 || n > (1ll << 31) - 1) return invalid("asicp: bad problem count");
  if (n > 0 && (!src_off || !ref_off || !thetas)) return invalid("asicp: null batch array");
  for (int64_t i = 0; i < n; ++i) {
    const int64_t ns = src_off[i + 1] - src_off[i], nr = ref_off[i + 1] - ref_off[i];
    if (ns < 0 || nr < 0) return invalid("asicp: decreasing cloud offsets");
    if (ns == 0 || nr == 0) return invalid("icp_closed_form_step: empty cloud");
    if (ns >= (1ll << 31) || nr >= (1ll << 31)) return invalid("asicp: cloud too large");
    const double* q = thetas + 7 * i + 3;
    const double n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
    if (!(std::abs(std::sqrt(n2) - 1.0) <= 1e-6)) return invalid("rotation_matrix: quaternion is not unit-norm");
  }
  if (n == 0) return ASICP_OK;
  REG_CUDA(cudaSetDevice(device_));
  if (!icp_) icp_ = new Dev();
  Dev& D = *icp_;
  const int64_t tot_src = src_off[n] - src_off[0], tot_ref = ref_off[n] - ref_off[0];
  std::vector<long long> so(n + 1), ro(n + 1);
  for (int64_t i = 0; i <= n; ++i) {
    so[i] = src_off[i] - src_off[0];
    ro[i] = ref_off[i] - ref_off[0];
  }
  REG_CUDA(D.src.ensure(tot_src * 24));
  REG_CUDA(D.ref.ensure(tot_ref * 24));
  REG_CUDA(D.src_off.ensure((n + 1) * 8));
  REG_CUDA(D.ref_off.ensure((n + 1) * 8));
  REG_CUDA(D.cand.ensure(tot_ref * sizeof(float4)));
  REG_CUDA(D.geo.ensure(n * 32));
  REG_CUDA(D.init.ensure(n * 56));
  REG_CUDA(D.theta.ensure(n * 56));
  REG_CUDA(D.fy.ensure(tot_src * 4));
  REG_CUDA(D.status.ensure(n * 4));
  REG_CUDA(cudaMemcpyAsync(D.src.p, sources + 3 * src_off[0], tot_src * 24, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.ref.p, references + 3 * ref_off[0], tot_ref * 24, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.src_off.p, so.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.ref_off.p, ro.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st_));
  REG_CUDA(cudaMemcpyAsync(D.init.p, thetas, n * 56, cudaMemcpyHostToDevice, st_));
  reg_cand_kernel<<<static_cast<unsigned>(n), 256, 0, st_>>>(static_cast<const double*>(D.ref.p),
                                                             static_cast<const long long*>(D.ref_off.p),
                                                             static_cast<float4*>(D.cand.p),
                                                             static_cast<double*>(D.geo.p));
  IcpArgs a;
  a.src = static_cast<const double*>(D.src.p);
  a.src_off = static_cast<const long long*>(D.src_off.p);
  a.ref = static_cast<const double*>(D.ref.p);
  a.ref_off = static_cast<const long long*>(D.ref_off.p);
  a.cand = static_cast<const float4*>(D.cand.p);
  a.geo = static_cast<const double*>(D.geo.p);
  a.theta = static_cast<const double*>(D.init.p);
  a.match = static_cast<int*>(D.fy.p);
  a.out = static_cast<double*>(D.theta.p);
  a.degenerate = static_cast<int*>(D.status.p);
  icp_step_kernel<<<static_cast<unsigned>(n), 256, 0, st_>>>(a);
  REG_CUDA(cudaGetLastError());
  std::vector<double> th(7 * n);
  std::vector<int> dg(n);
  REG_CUDA(cudaMemcpyAsync(th.data(), D.theta.p, n * 56, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(dg.data(), D.status.p, n * 4, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaStreamSynchronize(st_));
  for (int64_t i = 0; i < n; ++i) {
    std::memcpy(out[i].theta, &th[7 * i], 56);
    out[i].degenerate = dg[i];
  }
  return ASICP_OK;
}

int RegBatch::run(asicp_registration* out, std::string* err) {
  if (!d_) {
    *err = "asicp: no registration batch prepared";
    return ASICP_INVALID_ARGUMENT;
  }
  Dev& D = *d_;
  kernel_ms_ = 0.0f;
  if (D.n == 0) return ASICP_OK;
  REG_CUDA(cudaSetDevice(device_));
  RegArgs a;
  a.src = static_cast<const double*>(D.src.p);
  a.src_off = static_cast<const long long*>(D.src_off.p);
  a.ref = static_cast<const double*>(D.ref.p);
  a.ref_off = static_cast<const long long*>(D.ref_off.p);
  a.cand = static_cast<const float4*>(D.cand.p);
  a.cand_off = static_cast<const long long*>(D.ref_off.p);
  a.geo = static_cast<const double*>(D.geo.p);
  a.init = static_cast<const double*>(D.init.p);
  a.seeds = static_cast<const unsigned long long*>(D.seeds.p);
  a.fy_global = static_cast<int*>(D.fy.p);
  a.bat_global = static_cast<int*>(D.bat.p);
  a.theta = static_cast<double*>(D.theta.p);
  a.iters = static_cast<long long*>(D.iters.p);
  a.loss = static_cast<double*>(D.loss.p);
  a.conv = static_cast<int*>(D.conv.p);
  a.status = static_cast<int*>(D.status.p);
  // ASICP_REG_PROFILE=1: per-phase clocks of problem 0 to stderr (diagnostics).
  const bool prof = std::getenv("ASICP_REG_PROFILE") != nullptr;
  a.prof = nullptr;
  if (prof) {
    REG_CUDA(D.prof.ensure(32 * 8));
    REG_CUDA(cudaMemsetAsync(D.prof.p, 0, 32 * 8, st_));
    a.prof = static_cast<unsigned long long*>(D.prof.p);
  }
  a.ref_cap = D.ref_cap;
  a.fy_cap = D.fy_cap;
  a.bat_cap = D.bat_cap;
  a.pts_cap = D.pts_cap;
  a.pts_off = D.pts_off;
  REG_CUDA(cudaEventRecord(D.ev0, st_));
  register_kernel<<<D.n, kRegThreads, D.smem, st_>>>(a, D.cfg);
  REG_CUDA(cudaGetLastError());
  REG_CUDA(cudaEventRecord(D.ev1, st_));
  const size_t n = static_cast<size_t>(D.n);
  REG_CUDA(cudaMemcpyAsync(D.h_theta, D.theta.p, n * 56, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(D.h_iters, D.iters.p, n * 8, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(D.h_loss, D.loss.p, n * 8, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(D.h_conv, D.conv.p, n * 4, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaMemcpyAsync(D.h_status, D.status.p, n * 4, cudaMemcpyDeviceToHost, st_));
  REG_CUDA(cudaStreamSynchronize(st_));
  REG_CUDA(cudaEventElapsedTime(&kernel_ms_, D.ev0, D.ev1));
  if (prof) {
    unsigned long long h[32];
    REG_CUDA(cudaMemcpy(h, D.prof.p, sizeof h, cudaMemcpyDeviceToHost));
    const char* names[14] = {"iter-start", "nn-scan", "B-wait", "accumulate", "divide",
                             "parallel-tail", "thread0-tail", "final-barrier", "drawer-pre", "draw",
                             "B-merge", "B-resolve", "B-terms", "A-setup"};
    const double it = h[14] ? static_cast<double>(h[14]) : 1.0;
    for (int i = 0; i < 14; ++i)
      std::fprintf(stderr, "reg-phase %-14s worker %9.0f drawer %9.0f cycles/iter\n", names[i], h[i] / it,
                   h[16 + i] / it);
  }
  for (size_t i = 0; i < n; ++i) {
    if (D.h_status[i]) {
      *err = "rotation_matrix: quaternion is not unit-norm";
      return ASICP_INVALID_ARGUMENT;
    }
  }
  if (out)
    for (size_t i = 0; i < n; ++i) {
      std::memcpy(out[i].theta, D.h_theta + 7 * i, 56);
      out[i].iterations = D.h_iters[i];
      out[i].final_loss = D.h_loss[i];
      out[i].converged = D.h_conv[i];
    }
  return ASICP_OK;
}

double run_dfma_peak(int iters) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8;
  dfma_peak_kernel<<<blocks, 256>>>(out, iters / 4, 0.999, 1e-4);  // warm-up
  cudaEventRecord(e0);
  dfma_peak_kernel<<<blocks, 256>>>(out, iters, 0.999, 1e-4);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess || ms <= 0.0f) return -1.0;
  return 2.0 * 8.0 * static_cast<double>(iters) * blocks * 256.0 / (ms * 1e-3) / 1e12;
}

}  // namespace asicp
