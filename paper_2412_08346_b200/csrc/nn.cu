// Certified brute-force nearest neighbour (NN) on B200 — the hot loop of
// optimize_grasp: the forward match of match_surface_to_pool
// (grasp.cpp:92-106), the reverse match of collision_loss_and_gradients
// (grasp.cpp:68-84) and the final full-cloud ranking (grasp.cpp:263-281),
// replacing the per-call kd-trees of spatial_index.cpp:14-105.
//
// FP32 filter, FP64 decision:
//   * forward / final work item: (particle, <= 1024 queries, a split of the
//     candidates); the number of splits is picked on the device per round
//     (fwd_split) so that few matching particles still fill the grid; a split
//     is consumed in sub-chunks of <= 2048 candidates loaded whole into shared
//     memory by TMA bulk copies (cp.async.bulk + mbarrier, one 4 KB tile per
//     stage) and read with broadcast LDS.128;
//   * each thread holds 8 queries in registers; candidates are stored
//     pair-interleaved so one packed FFMA2 evaluates the expansion form
//     |b|^2 - 2 a.b for two candidates (3 FFMA2 per 2 pairs + a 3-input
//     min), branch-free;
//   * every 32 candidates (a subtile) each query folds the subtile minimum into
//     a running top-3 of subtile minima (b1 <= b2 <= b3, subtiles s1, s2);
//   * after a sub-chunk, the reference's answer within it — min FP64
//     (p - q).squaredNorm(), ties to the lowest position (spatial_index.cpp:
//     69-83) — is provably in {d32 <= b1 + 2E} (2E = the query's margin).  The
//     subtiles s1 (and s2 when b2 is inside the margin) are rescanned from
//     shared memory for the position of b1 and the window members;
//   * the running (best value, position) state carries across sub-chunks; a
//     window of one is certified, larger windows keep their members in a
//     pooled list and are decided in FP64 with the reference formula (after
//     the split merge); overflowing windows take a full FP64 rescan;
//   * reverse match: warp items (nn_rev_kernel, below).
#include "common.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace asicp {

constexpr int kFwdQ = 8;                     // forward / final: 8 queries per thread
constexpr int kFwdQB = kNnThreads * kFwdQ;   // queries per forward item
constexpr int kNnSmem = kNnStages * kNnTile * 16;
constexpr int kMinChunk = 2 * kNnTile;       // smallest candidate split

// ---------------------------------------------------------------------------
// Work planning: per particle counts -> exclusive scans -> item lists, all
// in nn_fill_kernel.
// Forward: count = query blocks; the split factor is chosen on the device
// from the total T so that T x splits ~ plan.target_items (few matching
// particles -> many splits per particle), capped by plan.nchunks and by
// kMinChunk candidates per split.  Reverse: warp items of kRevWQ points.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void fwd_split(int T, const NnPlan& plan, int* nch_out, int* chunk_out) {
  const int nmax = T > 0 ? max(1, min(plan.nchunks, min(plan.m / kMinChunk, ceil_div(plan.target_items, T)))) : 1;
  // Among 1..nmax splits, the one with the shortest estimated makespan on the
  // persistent grid (target_items / 4 CTAs): rounds of items x (candidates
  // per item + a per-item overhead), so the last round of equal items is as
  // full as it can be.  T x splits <= target_items keeps the item lists in
  // their preallocated size.
  // Throughput mode (contexts that share the GPU, batch.py): other solves
  // fill a round's idle CTAs, so only the per-item cost of full rounds counts.
  // Latency mode (one solve alone): list-scheduling makespan — the work spread
  // over every CTA slot plus the last item's length.
  const int grid = max(1, plan.target_items / 4);
  int nch = nmax;
  if (plan.use_tc) {
    // Tensor-core filter: every item is 8 units of 128 queries on one CTA
    // per SM; split only as far as needed for about target_items / 2 units
    // (each unit boundary costs a pipeline refill).
    nch = max(1, min(nmax, ceil_div(plan.target_items / 2, 8 * max(T, 1))));
    const int chunk = round_up(ceil_div(plan.m, nch), kNnTile);
    *chunk_out = chunk;
    *nch_out = ceil_div(plan.m, chunk);
    return;
  }
  long long best = -1;
  for (int s = 1; s <= nmax; ++s) {
    const int chunk = round_up(ceil_div(plan.m, s), kNnTile);
    const int items = T * ceil_div(plan.m, chunk);
    const long long per = chunk + plan.item_overhead;
    const long long cost = plan.throughput ? static_cast<long long>(ceil_div(items, grid)) * per
                                           : static_cast<long long>(items) * per / grid + per;
    if (best < 0 || cost < best) {  // ties: fewer splits (less merging)
      best = cost;
      nch = s;
    }
  }
  const int chunk = round_up(ceil_div(plan.m, nch), kNnTile);
  *chunk_out = chunk;
  *nch_out = ceil_div(plan.m, chunk);
}

// Item counts of particle j: forward query blocks, or reverse warp items when
// the particle collides (the final ranking matches every particle forward).
__device__ __forceinline__ void plan_counts(const DevProblem& P, const DevState& S, const NnPlan& plan, int j,
                                            int* fwd, int* rev) {
  *fwd = *rev = 0;
  if (plan.kind == 2 || S.active[j]) {
    if (plan.kind != 2 && S.n_col[j] > 0)
      *rev = ceil_div(S.n_col[j], kRevWQ);
    else
      *fwd = ceil_div(surf_count(P, j), kFwdQB);
  }
}

// Planning and item fill in one launch: every CTA recomputes the exclusive
// scans of the per-particle counts (a few hundred to a few thousand
// particles — cheaper than a second launch and a one-CTA kernel), then fills
// the items of its own 128 particles; CTA 0 publishes the totals and resets
// the round's counters.
constexpr int kFillThreads = 128;
__global__ void __launch_bounds__(kFillThreads) nn_fill_kernel(DevProblem P, DevState S, NnPlan plan) {
  pdl_enter();
  __shared__ int sf[kFillThreads], sr[kFillThreads];
  const int tid = threadIdx.x;
  const int per = ceil_div(P.J, kFillThreads);
  {
    const int j0 = min(P.J, tid * per), j1 = min(P.J, j0 + per);
    int cf = 0, cr = 0;
    for (int jj = j0; jj < j1; ++jj) {
      int f, r;
      plan_counts(P, S, plan, jj, &f, &r);
      cf += f;
      cr += r;
    }
    sf[tid] = cf;
    sr[tid] = cr;
  }
  __syncthreads();
  for (int off = 1; off < kFillThreads; off <<= 1) {  // inclusive scans of the range sums
    const int vf = tid >= off ? sf[tid - off] : 0, vr = tid >= off ? sr[tid - off] : 0;
    __syncthreads();
    sf[tid] += vf;
    sr[tid] += vr;
    __syncthreads();
  }
  const int T = sf[kFillThreads - 1];
  if (blockIdx.x == 0 && tid == 0) {
    S.item_off[0][P.J] = T;
    S.item_off[1][P.J] = sr[kFillThreads - 1];
    S.item_count[0][P.J] = S.item_count[1][P.J] = 0;
    S.item_counter[0] = S.item_counter[1] = 0;
    *S.refine_count = 0;
    *S.amb_count = 0;
  }
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.J) return;
  {
    // Offsets of j: the scan up to its range, plus the counts before j in it.
    const int r = j / per;
    int of = r ? sf[r - 1] : 0, orr = r ? sr[r - 1] : 0;
    for (int jj = r * per; jj < j; ++jj) {
      int f, rv;
      plan_counts(P, S, plan, jj, &f, &rv);
      of += f;
      orr += rv;
    }
    int f, rv;
    plan_counts(P, S, plan, j, &f, &rv);
    S.item_count[0][j] = f;
    S.item_count[1][j] = rv;
    S.item_off[0][j] = of;
    S.item_off[1][j] = orr;
  }
  int nch, chunk;
  fwd_split(T, plan, &nch, &chunk);
  if (j == 0) {
    S.nn_dyn[0] = nch;
    S.nn_dyn[1] = T * nch;
  }
  const int64_t so = P.part_surf_off[j];
  const int ns = surf_count(P, j);
  if (S.item_count[1][j] > 0) {
    const int nq = S.n_col[j];
    const int64_t row = static_cast<int64_t>(j) * P.n_scene;
    int w = S.item_off[1][j];
    for (int b = 0; b < S.item_count[1][j]; ++b) {
      NnItem it;
      it.q = S.col_q + row + b * kRevWQ;
      it.nq = min(kRevWQ, nq - b * kRevWQ);
      it.c = S.Sc32 + so;
      it.nc = ns;
      it.c_base = 0;
      it.kind = 1;
      it.owner = j;
      it.q_first = b * kRevWQ;
      it.chunk = 0;
      it.nchunks = 1;
      it.slot = 0;
      S.items[1][w++] = it;
    }
  }
  if (S.item_count[0][j] > 0) {
    const float4* cands = plan.pooled ? S.pool32 + static_cast<int64_t>(j) * P.n_obj_pad : P.obj_cand;
    const int qb0 = S.item_off[0][j];
    for (int b = 0; b < S.item_count[0][j]; ++b)
      for (int s = 0; s < nch; ++s) {
        NnItem it;
        it.q = S.Sq32 + so + b * kFwdQB;
        it.nq = min(kFwdQB, ns - b * kFwdQB);
        const int c0 = s * chunk;
        it.c = cands + c0;
        it.nc = min(chunk, plan.m - c0);
        it.c_base = c0;
        it.kind = plan.kind;
        it.owner = j;
        it.q_first = b * kFwdQB;
        it.chunk = s;
        it.nchunks = nch;
        it.slot = qb0 + b;
        S.items[0][(qb0 + b) * nch + s] = it;
      }
  }
}

// ---------------------------------------------------------------------------
// FP64 decision with the reference formula.
// ---------------------------------------------------------------------------
struct NnGeom {
  const double* qpt;     // query point (FP64)
  const double* cbase;   // candidate FP64 rows
  const int* cmap;       // candidate position -> row (minibatch pool), or null
};

__device__ __forceinline__ NnGeom nn_geom(const DevProblem& P, const DevState& S, const NnPlan& plan, int kind,
                                          int j, int qlocal) {
  NnGeom g;
  const int64_t so = P.part_surf_off[j];
  if (kind == 1) {
    const int64_t row = static_cast<int64_t>(j) * P.n_scene;
    g.qpt = P.scene64 + 3 * static_cast<int64_t>(S.col_idx[row + qlocal]);
    g.cbase = S.S64 + 3 * so;
    g.cmap = nullptr;
  } else {
    g.qpt = S.S64 + 3 * (so + qlocal);
    g.cbase = P.obj64;
    g.cmap = (kind == 0 && plan.pooled) ? S.pool_idx + static_cast<int64_t>(j) * P.n_obj_pad : nullptr;
  }
  return g;
}

// spatial_index.cpp:69: (points[idx] - query).squaredNorm()
__device__ __forceinline__ double nn_d64(const NnGeom& g, int pos) {
  const int64_t r = g.cmap ? g.cmap[pos] : pos;
  const V3 p = load3(g.cbase, r);
  return sqnorm(sub(p, V3{g.qpt[0], g.qpt[1], g.qpt[2]}));
}

__device__ __forceinline__ int* nn_result_slot(const DevProblem& P, const DevState& S, int kind, int j, int qlocal) {
  if (kind == 1) return S.res_rev + static_cast<int64_t>(j) * P.n_scene + qlocal;
  return S.res_fwd + P.part_surf_off[j] + qlocal;
}

// Window decision: strictly closer wins, equal distance -> lowest position.
// Exact ties between distinct rows of a canonical-order forward set are
// counted (the reference would break them by its sampled pool order).
__device__ __forceinline__ int nn_decide(const NnGeom& g, const int* pos, int n, bool tie_sensitive,
                                         unsigned long long* stats) {
  if (n == 1) return pos[0];
  atomicAdd(stats + 0, 1ull);
  double best = 0.0;
  int bi = -1;
  bool tie = false;
  for (int e = 0; e < n; ++e) {
    const double d = nn_d64(g, pos[e]);
    if (bi >= 0 && d == best) tie = true;
    if (bi < 0 || d < best || (d == best && pos[e] < bi)) {
      if (bi < 0 || d < best) tie = false;
      best = d;
      bi = pos[e];
    }
  }
  if (tie && tie_sensitive) atomicAdd(stats + 3, 1ull);
  return bi;
}

// Ambiguous-window member lists: a block of kWinCap (position, d32) entries
// per ambiguous query, allocated from a pool; amb_n > kWinCap marks overflow.
__device__ __forceinline__ int win_alloc(const DevState& S) {
  const int b = atomicAdd(S.amb_count, 1);
  return b < S.amb_cap ? b : -1;
}
__device__ __forceinline__ void win_push(const DevState& S, int blk, int pos, float d) {
  const int n = S.amb_n[blk];
  if (n < kWinCap) S.amb_pool[static_cast<int64_t>(blk) * kWinCap + n] = make_int2(pos, __float_as_int(d));
  S.amb_n[blk] = n + 1;
}
// Members of a running window with d32 <= thr; false if they cannot be listed.
__device__ __forceinline__ bool win_collect(const DevState& S, int p1, float thr, int* out, int* n, int cap) {
  if (!(p1 & kAmbiguous)) {
    if (cap < 1) return false;
    out[0] = p1;
    *n = 1;
    return true;
  }
  const int blk = p1 & ~kAmbiguous;
  if (blk == kNoBlock) return false;
  const int cnt = S.amb_n[blk];
  if (cnt > kWinCap) return false;
  int m = 0;
  for (int e = 0; e < cnt; ++e) {
    const int2 v = S.amb_pool[static_cast<int64_t>(blk) * kWinCap + e];
    if (__int_as_float(v.y) <= thr) {
      if (m >= cap) return false;
      out[m++] = v.x;
    }
  }
  *n = m;
  return m > 0;
}

// stats[5 + kind]: rescans per match kind; stats[8 + reason]: 0 validation
// mode, 1 ambiguous window, 3 ambiguous across splits; stats[16 + k]: rescans
// in iteration k.
__device__ __forceinline__ void push_refine(const DevState& S, int kind, int j, int qlocal, int reason, int iter) {
  const int slot = atomicAdd(S.refine_count, 1);
  if (slot < S.refine_cap) S.refine_list[slot] = make_int4(kind, j, qlocal, 0);
  atomicAdd(S.stats + 1, 1ull);
  atomicAdd(S.stats + 5 + kind, 1ull);
  atomicAdd(S.stats + 8 + reason, 1ull);
  atomicAdd(S.stats + 16 + min(iter, 223), 1ull);
}

// ---------------------------------------------------------------------------
// TMA / mbarrier primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float d32(float qx, float qy, float qz, float4 v) {
  return __fmaf_rn(qx, v.x, __fmaf_rn(qy, v.y, __fmaf_rn(qz, v.z, v.w)));
}

// Packed FP32 pairs (sm_100 FFMA2): two queries share one instruction; a
// scalar candidate operand is broadcast to both lanes (ptxas folds the
// {v, v} pair into a .F32 broadcast operand).  Each lane is an IEEE fma, so
// the values equal d32() bit for bit.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(f32x2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float half2f(f32x2 v, int k) {
  float lo, hi;
  up2(v, lo, hi);
  return (k & 1) ? hi : lo;
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// Running window of one query (position / ambiguous-list state).
struct RunState {
  float b;
  int p;
};

// Sub-chunk epilogue of one query, out of line: the kernel keeps one copy of
// this code instead of Q unrolled ones.  At small candidate counts (early
// minibatch iterations) the instruction fetch of the unrolled copies, not the
// arithmetic, set the launch time.  Members of the sub-chunk's window and the
// position of its minimum are merged into the running window (an explicit
// member list only once it holds two).
__device__ __noinline__ RunState subchunk_window(const DevState& S, const float4* tiles, int base, float qx,
                                                 float qy, float qz, float b1, float b2, float b3, int s12, float mg,
                                                 RunState run) {
  RunState out = run;
  {
        const float thr = __fadd_ru(b1, mg);
        bool ovf = b3 <= thr;
        int pmin = -1, np = 0;
        int mpos[kWinCap];
        float md[kWinCap];
        const int nscan = b2 <= thr ? 2 : 1;
        // Window members of the best one or two subtiles: a member bitmask
        // from one pass of shared-memory loads (the tiles are shared; this
        // out-of-line function sees a generic pointer, hence ld.shared by
        // address), then the members in increasing position.
        const uint32_t tiles_s = static_cast<uint32_t>(__cvta_generic_to_shared(tiles));
        for (int r = 0; r < nscan; ++r) {
          const int sid = r == 0 ? (s12 & 0xffff) : (s12 >> 16);
          const uint32_t sp = tiles_s + static_cast<uint32_t>(sid * kSub) * 16u;
          unsigned mask = 0;
#pragma unroll
          for (int c = 0; c < kSub; c += 2) {
            // One interleaved pair (two 16-byte loads): candidates c and c + 1,
            // evaluated together by packed FMAs (each lane is d32()).
            const float4 A = lds128(sp + c * 16u), B = lds128(sp + (c + 1) * 16u);
            f32x2 d = ffma2(pk2(B.x, B.y), pk2(qz, qz), pk2(B.z, B.w));
            d = ffma2(pk2(A.z, A.w), pk2(qy, qy), d);
            d = ffma2(pk2(A.x, A.y), pk2(qx, qx), d);
            float d0, d1;
            up2(d, d0, d1);
            if (d0 <= thr) mask |= 1u << c;
            if (d1 <= thr) mask |= 1u << (c + 1);
          }
          while (mask) {
            const int c = __ffs(mask) - 1;
            mask &= mask - 1;
            const uint32_t cp = static_cast<uint32_t>(c & ~1);
            const float4 A = lds128(sp + cp * 16u), B = lds128(sp + (cp + 1) * 16u);
            const float d = (c & 1) ? d32(qx, qy, qz, make_float4(A.y, A.w, B.y, B.w))
                                    : d32(qx, qy, qz, make_float4(A.x, A.z, B.x, B.z));
            const int p = base + sid * kSub + c;
            if (np < kWinCap) {
              mpos[np] = p;
              md[np] = d;
            }
            ++np;
            if (d == b1 && (pmin < 0 || p < pmin)) pmin = p;
          }
        }
        ovf = ovf || np > kWinCap;
        const float run_b = run.b;
        const int run_p = run.p;
        if (b1 < run_b) {
          // New best: old members stay in the window only if the old best is
          // still within the new margin.
          const bool keep_old = run_b <= thr;
          if (!keep_old && np == 1 && !ovf) {
            out.p = pmin;
          } else {
            // The running window is certified (run_p a position), listed (a
            // block of the pool) or listless (the pool ran out: kNoBlock).  A
            // listless window that stays inside the new margin keeps the query
            // listless; otherwise a fresh block takes the new members.
            const bool was_amb = (run_p & kAmbiguous) != 0;
            const bool old_listed = was_amb && (run_p & ~kAmbiguous) != kNoBlock;
            int blk = -1;
            if (old_listed)
              blk = run_p & ~kAmbiguous;
            else if (!(was_amb && keep_old))
              blk = win_alloc(S);
            if (blk >= 0) {
              if (!old_listed) {
                S.amb_n[blk] = 0;
                if (keep_old) win_push(S, blk, run_p, run_b);  // certified old best (was_amb is false here)
              } else if (!keep_old) {
                S.amb_n[blk] = 0;
              }
              for (int e = 0; e < min(np, kWinCap); ++e) win_push(S, blk, mpos[e], md[e]);
              if (ovf) S.amb_n[blk] = kWinCap + 1;
            }
            out.p = kAmbiguous | (blk >= 0 ? blk : kNoBlock);
          }
          out.b = b1;
        } else if (b1 <= __fadd_ru(run_b, mg)) {
          const float run_thr = __fadd_ru(run_b, mg);
          int blk = (run_p & kAmbiguous) ? (run_p & ~kAmbiguous) : win_alloc(S);
          if (blk >= 0 && blk != kNoBlock) {
            if (!(run_p & kAmbiguous)) {
              S.amb_n[blk] = 0;
              win_push(S, blk, run_p, run_b);
            }
            for (int e = 0; e < min(np, kWinCap); ++e)
              if (md[e] <= run_thr) win_push(S, blk, mpos[e], md[e]);
            if (ovf) S.amb_n[blk] = kWinCap + 1;
          }
          out.p = kAmbiguous | (blk >= 0 ? blk : kNoBlock);
        }
      }
  return out;
}

// Emit of an ambiguous query (out of line, see subchunk_window): decide the
// window members in FP64 with the reference formula, or queue a full rescan.
__device__ __noinline__ void emit_ambiguous(const DevProblem& P, const DevState& S, const NnPlan& plan, int kind,
                                            int owner, int qlocal, int p1, float thr) {
  int pos[kWinCap];
  int n = 0;
  if (win_collect(S, p1, thr, pos, &n, kWinCap)) {
    const NnGeom g = nn_geom(P, S, plan, kind, owner, qlocal);
    *nn_result_slot(P, S, kind, owner, qlocal) = nn_decide(g, pos, n, kind == 0 && !plan.pooled, S.stats);
  } else {
    push_refine(S, kind, owner, qlocal, 1, plan.iter);
  }
}

// ---------------------------------------------------------------------------
// The filter kernel (persistent over one work list).
// ---------------------------------------------------------------------------
// 4 CTAs (16 warps) per SM: with the packed FFMA2 main loop the kernel fits
// 128 registers without spilling, and the extra warps hide the FFMA2 / LDS
// latencies that stall a 2-CTA configuration.
// -DASICP_NN_PHASES: per-warp clock() accounting of the filter's phases
// (diagnostic build; tools/nn_phases.sh), summed into stats[240 + phase].
#ifdef ASICP_NN_PHASES
#define NNPH_DECL unsigned int ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; unsigned int ph_t = clock();
#define NNPH(i)                        \
  {                                    \
    const unsigned int ph_now = clock(); \
    ph_acc[i] += ph_now - ph_t;        \
    ph_t = ph_now;                     \
  }
#define NNPH_FLUSH                                                                               \
  if ((threadIdx.x & 31) == 0)                                                                   \
    for (int i_ = 0; i_ < 8; ++i_) atomicAdd(S.stats + 240 + i_, static_cast<unsigned long long>(ph_acc[i_]));
#else
#define NNPH_DECL
#define NNPH(i)
#define NNPH_FLUSH
#endif

template <int Q>
#ifndef ASICP_NN_MINBLOCKS
#define ASICP_NN_MINBLOCKS 4
#endif
__global__ void __launch_bounds__(kNnThreads, ASICP_NN_MINBLOCKS)
    nn_filter_kernel(const __grid_constant__ DevProblem P, const __grid_constant__ DevState S,
                     const __grid_constant__ NnPlan plan, int list) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float4* tiles = reinterpret_cast<float4*>(smem_raw);
  __shared__ __align__(8) uint64_t full_bar[kNnStages];
  __shared__ int s_item;
  __shared__ float run_mg[Q * kNnThreads];
  __shared__ float run_b1[Q * kNnThreads];
  __shared__ int run_p1[Q * kNnThreads];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kNnStages; ++s) mbar_init(&full_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_items = list == 0 ? S.nn_dyn[1] : S.item_off[list][P.J];
  const NnItem* items = S.items[list];
  uint32_t phases = 0;  // bit s: parity of the next completion of stage s
  NNPH_DECL
  for (;;) {
    if (tid == 0) s_item = atomicAdd(S.item_counter + list, 1);
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= n_items) break;
    const NnItem w = items[it];
    if (tid == 0) {
      atomicAdd(S.stats + 2, static_cast<unsigned long long>(w.chunk == 0 ? w.nq : 0));
      atomicAdd(S.stats + 4, static_cast<unsigned long long>(w.nq) * static_cast<unsigned long long>(w.nc));
      if (list == 0)
        atomicAdd(S.stats + 12, static_cast<unsigned long long>(w.nq) * static_cast<unsigned long long>(w.nc));
      unsigned long long* is = S.iter_stats + 4 * plan.iter + list;
      atomicAdd(is, static_cast<unsigned long long>(w.nq) * static_cast<unsigned long long>(w.nc));
      if (w.chunk == 0) atomicAdd(is + 2, static_cast<unsigned long long>(w.nq));
    }
    // Running state lives in shared memory (touched once per sub-chunk), which
    // keeps the hot loop's register footprint down.
    float qx[Q], qy[Q], qz[Q];
#define MG(k) run_mg[(k) * kNnThreads + tid]
#define B1(k) run_b1[(k) * kNnThreads + tid]
#define P1(k) run_p1[(k) * kNnThreads + tid]
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const int qi = tid + k * kNnThreads;
      const float4 q = qi < w.nq ? w.q[qi] : make_float4(0.f, 0.f, 0.f, 0.f);
      qx[k] = q.x;
      qy[k] = q.y;
      qz[k] = q.z;
      MG(k) = q.w;
      B1(k) = INFINITY;
      P1(k) = 0;
    }
    for (int sc0 = 0; sc0 < w.nc; sc0 += kNnMaxChunk) {
      const int nsc = min(kNnMaxChunk, w.nc - sc0);
      const int nsc_pad = round_up(nsc, kSub);  // candidate arrays are padded with +inf rows
      const int ntiles = ceil_div(nsc_pad, kNnTile);
      if (tid == 0) {
        for (int t = 0; t < ntiles; ++t) {
          const int n_in = min(kNnTile, nsc_pad - t * kNnTile);
          tma_load_1d(tiles + t * kNnTile, w.c + sc0 + t * kNnTile, n_in * 16, &full_bar[t]);
        }
      }
      float b1[Q], b2[Q], b3[Q];
      int s1v[Q], s2v[Q];
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        b1[k] = b2[k] = b3[k] = INFINITY;
        s1v[k] = s2v[k] = 0;
      }
      NNPH(0)
      for (int t = 0; t < ntiles; ++t) {
        mbar_wait(&full_bar[t], (phases >> t) & 1u);
        phases ^= 1u << t;
        NNPH(1)
        const float4* tile = tiles + t * kNnTile;
        const int nsub = min(kNnTile, nsc_pad - t * kNnTile) / kSub;
        for (int sub = 0; sub < nsub; ++sub) {
          const float4* sp = tile + sub * kSub;
          float tm[Q];
#pragma unroll
          for (int k = 0; k < Q; ++k) tm[k] = INFINITY;
          // Candidates are pair-interleaved (pc_index): one LDS.128 gives the
          // (x0, x1, y0, y1) pairs, the next (z0, z1, w0, w1).  Each packed
          // FFMA2 evaluates two candidates for one query (query coordinate
          // broadcast); per lane the arithmetic is d32():
          // fma(qx,vx, fma(qy,vy, fma(qz,vz, w))).  Four candidates per step,
          // each FMA stage issued across all Q queries before the next.
#pragma unroll  // the whole subtile: 0.60 of the FMA pipe vs 0.57 at 2 steps (tools/nn_loop_bench.cu)
          for (int c = 0; c < kSub; c += 4) {
            const float4 a0 = sp[c], c0 = sp[c + 1];  // candidates c, c+1
            const float4 a1 = sp[c + 2], c1 = sp[c + 3];  // candidates c+2, c+3
            const f32x2 x0 = pk2(a0.x, a0.y), y0 = pk2(a0.z, a0.w), z0 = pk2(c0.x, c0.y), w0 = pk2(c0.z, c0.w);
            const f32x2 x1 = pk2(a1.x, a1.y), y1 = pk2(a1.z, a1.w), z1 = pk2(c1.x, c1.y), w1 = pk2(c1.z, c1.w);
            f32x2 d0[Q], d1[Q];
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              d0[k] = ffma2(z0, pk2(qz[k], qz[k]), w0);
              d1[k] = ffma2(z1, pk2(qz[k], qz[k]), w1);
            }
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              d0[k] = ffma2(y0, pk2(qy[k], qy[k]), d0[k]);
              d1[k] = ffma2(y1, pk2(qy[k], qy[k]), d1[k]);
            }
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              d0[k] = ffma2(x0, pk2(qx[k], qx[k]), d0[k]);
              d1[k] = ffma2(x1, pk2(qx[k], qx[k]), d1[k]);
            }
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              float l0, h0, l1, h1;
              up2(d0[k], l0, h0);
              up2(d1[k], l1, h1);
              tm[k] = fminf(fminf(tm[k], fminf(l0, h0)), fminf(l1, h1));
            }
          }
          NNPH(2)
          const int sid = t * (kNnTile / kSub) + sub;
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            // Running top-3 of subtile minima as a min/max network (equal
            // values keep the earlier subtile: positions move on strict <).
            const bool lt1 = tm[k] < b1[k];
            const bool lt2 = tm[k] < b2[k];
            b3[k] = fminf(b3[k], fmaxf(b2[k], tm[k]));
            b2[k] = fminf(b2[k], fmaxf(b1[k], tm[k]));
            b1[k] = fminf(b1[k], tm[k]);
            s2v[k] = lt1 ? s1v[k] : (lt2 ? sid : s2v[k]);
            s1v[k] = lt1 ? sid : s1v[k];
          }
          NNPH(3)
        }
      }
      // Sub-chunk epilogue (candidates still resident): members of the
      // sub-chunk's window and the position of its minimum, merged into the
      // running window (an explicit member list only once it holds two).
      // Common case, inline for all Q queries at once: a new best (b1 below
      // the running best, which falls outside the new window) whose window
      // lies in subtile s1 alone (b2 outside it) and holds one member — the
      // certified position.  Anything else takes subchunk_window; a sub-chunk
      // whose best is outside the running window leaves it unchanged.
      {
        const uint32_t tiles_s = static_cast<uint32_t>(__cvta_generic_to_shared(tiles));
        unsigned msk[Q];
        float thrv[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          thrv[k] = __fadd_ru(b1[k], MG(k));
          const uint32_t sp = tiles_s + static_cast<uint32_t>(s1v[k] * kSub) * 16u;
          unsigned m = 0;
#pragma unroll
          for (int c = 0; c < kSub; c += 2) {
            const float4 A = lds128(sp + c * 16u), B = lds128(sp + (c + 1) * 16u);
            f32x2 d = ffma2(pk2(B.x, B.y), pk2(qz[k], qz[k]), pk2(B.z, B.w));
            d = ffma2(pk2(A.z, A.w), pk2(qy[k], qy[k]), d);
            d = ffma2(pk2(A.x, A.y), pk2(qx[k], qx[k]), d);
            float d0, d1;
            up2(d, d0, d1);
            if (d0 <= thrv[k]) m |= 1u << c;
            if (d1 <= thrv[k]) m |= 1u << (c + 1);
          }
          msk[k] = m;
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const float run_b = B1(k), mg = MG(k);
          if (b1[k] > __fadd_ru(run_b, mg)) continue;  // cannot change the running window
          if (b1[k] < run_b && !(run_b <= thrv[k]) && b2[k] > thrv[k] && __popc(msk[k]) == 1) {
            B1(k) = b1[k];
            P1(k) = w.c_base + sc0 + s1v[k] * kSub + __ffs(msk[k]) - 1;
            continue;
          }
          const RunState r = subchunk_window(S, tiles, w.c_base + sc0, qx[k], qy[k], qz[k], b1[k], b2[k], b3[k],
                                             s1v[k] | (s2v[k] << 16), mg, RunState{run_b, P1(k)});
          B1(k) = r.b;
          P1(k) = r.p;
        }
      }
      NNPH(4)
      __syncthreads();  // all rescans done before the next sub-chunk overwrites the tiles
      NNPH(5)
    }
    // Emit.
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const int qi = tid + k * kNnThreads;
      if (qi >= w.nq) continue;
      const int qlocal = w.q_first + qi;
      const int p1 = P1(k);
      if (w.nchunks == 1) {
        if (plan.fp64_mode) {
          push_refine(S, w.kind, w.owner, qlocal, 0, plan.iter);
        } else if (!(p1 & kAmbiguous)) {
          *nn_result_slot(P, S, w.kind, w.owner, qlocal) = p1;  // certified
        } else {
          emit_ambiguous(P, S, plan, w.kind, w.owner, qlocal, p1, __fadd_ru(B1(k), MG(k)));
        }
      } else {
        NnPartial pr;
        pr.b1 = B1(k);
        pr.pos = p1;
        S.partials[(static_cast<int64_t>(w.slot) * w.nchunks + w.chunk) * kFwdQB + qi] = pr;
      }
    }
    NNPH(6)
  }
  NNPH(7)
  NNPH_FLUSH
}

// Merge the per-split results of forward/final queries (nchunks > 1): the
// global best is certified when exactly one split reaches the window and that
// split was itself unambiguous.
__global__ void nn_merge_kernel(DevProblem P, DevState S, NnPlan plan) {
  pdl_enter();
  const int j = blockIdx.y;
  const int nch = S.nn_dyn[0];
  if (nch <= 1) return;  // single split: the filter emitted directly
  if (plan.kind != 2 && (!S.active[j] || S.n_col[j] > 0)) return;
  const int64_t so = P.part_surf_off[j];
  const int ns = surf_count(P, j);
  const int qlocal = blockIdx.x * blockDim.x + threadIdx.x;
  if (qlocal >= ns) return;
  const NnPartial* parts =
      S.partials + static_cast<int64_t>(S.item_off[0][j] + qlocal / kFwdQB) * nch * kFwdQB + qlocal % kFwdQB;
  float b1 = INFINITY;
  int best = 0;
  for (int s = 0; s < nch; ++s) {
    const NnPartial p = parts[s * kFwdQB];
    if (p.b1 < b1) {
      b1 = p.b1;
      best = p.pos;
    }
  }
  if (plan.fp64_mode) {
    push_refine(S, plan.kind, j, qlocal, 0, plan.iter);
    return;
  }
  const float thr = __fadd_ru(b1, S.Sq32[so + qlocal].w);
  int reach = 0;
  for (int s = 0; s < nch; ++s) reach += parts[s * kFwdQB].b1 <= thr ? 1 : 0;
  if (reach == 1 && !(best & kAmbiguous)) {
    S.res_fwd[so + qlocal] = best;  // certified
    return;
  }
  // Gather every split's window members within the global window; decide in FP64.
  constexpr int kMax = 32;
  int pos[kMax];
  int n = 0;
  bool ok = true;
  for (int s = 0; s < nch && ok; ++s) {
    const NnPartial p = parts[s * kFwdQB];
    if (p.b1 > thr) continue;
    int m = 0;
    ok = win_collect(S, p.pos, thr, pos + n, &m, kMax - n) && ok;
    n += m;
  }
  if (!ok || n == 0) {
    push_refine(S, plan.kind, j, qlocal, 3, plan.iter);
    return;
  }
  const NnGeom g = nn_geom(P, S, plan, plan.kind, j, qlocal);
  S.res_fwd[so + qlocal] = nn_decide(g, pos, n, plan.kind == 0 && !plan.pooled, S.stats);
}

// Full FP64 rescan (ambiguous windows, and the FP64 validation mode): one
// warp per query, lexicographic (distance, position) minimum — exactly the
// reference's kd-tree rule.
// Full FP64 rescans (validation mode, overflowing or unlisted windows): one
// CTA per entry, every thread scanning a stride of the candidates with its
// loads batched (the candidate map and rows are L2 gathers), then a block
// argmin with the reference's tie rule (equal distance -> lowest position).
__global__ void __launch_bounds__(256) nn_refine_kernel(DevProblem P, DevState S, NnPlan plan) {
  pdl_enter();
  __shared__ double s_best[8];
  __shared__ int s_bi[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int total = min(*S.refine_count, S.refine_cap);
  for (int e = blockIdx.x; e < total; e += gridDim.x) {
    const int4 r = S.refine_list[e];
    const int kind = r.x, j = r.y, qlocal = r.z;
    const NnGeom g = nn_geom(P, S, plan, kind, j, qlocal);
    const int nc = kind == 1 ? surf_count(P, j) : plan.m;
    const V3 qp = V3{g.qpt[0], g.qpt[1], g.qpt[2]};
    double best = INFINITY;
    int bi = 0x7fffffff;
    constexpr int kU = 4;
    for (int c0 = threadIdx.x; c0 < nc; c0 += kU * blockDim.x) {
      int64_t row[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int c = c0 + u * blockDim.x;
        row[u] = c < nc ? (g.cmap ? g.cmap[c] : c) : 0;
      }
      V3 p[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) p[u] = load3(g.cbase, row[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int c = c0 + u * blockDim.x;
        if (c >= nc) continue;
        const double d = sqnorm(sub(p[u], qp));  // spatial_index.cpp:69
        if (d < best || (d == best && c < bi)) {
          best = d;
          bi = c;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) {
      s_best[wid] = best;
      s_bi[wid] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
        if (s_best[w] < best || (s_best[w] == best && s_bi[w] < bi)) {
          best = s_best[w];
          bi = s_bi[w];
        }
      *nn_result_slot(P, S, kind, j, qlocal) = bi;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Reverse match (collision_loss_and_gradients, grasp.cpp:68-84): each
// colliding scene point against the particle's transformed contact surface.
// Colliding points are few per particle (tens to hundreds), so a work item is
// <= kRevWQ points of one particle against its <= ~1k candidates, and the
// whole CTA works on one item: the surface is staged once into shared memory
// (cp.async, reused by the particle's next item), each warp scans every
// kRevWarps-th subtile for all the item's points (two per lane), and the
// per-warp top-3 subtile minima are merged in (value, subtile) order -- the
// same top-3 a single sequential scan keeps.  Same filter and certification
// as nn_filter_kernel with a single split: the window members are listed on
// the spot and decided in FP64 at once.
// ---------------------------------------------------------------------------
constexpr int kRevWarps = 4;
constexpr int kRevThreads = 32 * kRevWarps;
constexpr int kRevMaxC = 1024;  // candidates staged per CTA (16 KB); larger surfaces are read through L1
struct RevTop {
  float b1, b2, b3;
  int s1, s2;
};
constexpr int kRevSmem = kRevMaxC * 16 + kRevWarps * kRevWQ * static_cast<int>(sizeof(RevTop));
static int g_rev_blocks_per_sm = 1;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// (v, s) into a top-3 ordered by (value, subtile).
__device__ __forceinline__ void top3_insert(float& b1, int& s1, float& b2, int& s2, float& b3, float v, int s) {
  if (v < b1 || (v == b1 && s < s1)) {
    b3 = b2;
    b2 = b1;
    s2 = s1;
    b1 = v;
    s1 = s;
  } else if (v < b2 || (v == b2 && s < s2)) {
    b3 = b2;
    b2 = v;
    s2 = s;
  } else {
    b3 = fminf(b3, v);
  }
}

__global__ void __launch_bounds__(kRevThreads) nn_rev_kernel(DevProblem P, DevState S, NnPlan plan) {
  pdl_enter();
  extern __shared__ __align__(16) float4 rev_smem[];
  float4* stage = rev_smem;
  RevTop* tops = reinterpret_cast<RevTop*>(rev_smem + kRevMaxC);
  const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
  const int n_items = S.item_off[1][P.J];
  // Contiguous item ranges per CTA: a particle's items are consecutive, so
  // its surface is staged once.
  const int i0 = static_cast<int>(static_cast<long long>(blockIdx.x) * n_items / gridDim.x);
  const int i1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * n_items / gridDim.x);
  const float4* staged_c = nullptr;
  constexpr int QR = kRevWQ / 32;
  for (int it = i0; it < i1; ++it) {
    const NnItem w = S.items[1][it];
    const int ncp = round_up(w.nc, kSub);
    const bool staged = ncp <= kRevMaxC;
    __syncthreads();  // the previous item's epilogue is done with the stage and the tops
    if (staged && w.c != staged_c) {
      for (int c = tid; c < ncp; c += kRevThreads) cp_async16(stage + c, w.c + c);
      cp_async_wait_all();
      __syncthreads();
      staged_c = w.c;
    }
    const float4* cand = staged ? stage : w.c;
    if (tid == 0) {
      const unsigned long long pairs = static_cast<unsigned long long>(w.nq) * w.nc;
      atomicAdd(S.stats + 2, static_cast<unsigned long long>(w.nq));
      atomicAdd(S.stats + 4, pairs);
      atomicAdd(S.iter_stats + 4 * plan.iter + 1, pairs);
      atomicAdd(S.iter_stats + 4 * plan.iter + 3, static_cast<unsigned long long>(w.nq));
    }
    float4 q[QR];
#pragma unroll
    for (int r = 0; r < QR; ++r)
      q[r] = lane + 32 * r < w.nq ? w.q[lane + 32 * r] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int nsub = ceil_div(w.nc, kSub);  // candidate rows are +inf padded to the subtile
    float b1[QR], b2[QR], b3[QR];
    int s1[QR], s2[QR];
    f32x2 qx2[QR], qy2[QR], qz2[QR];
#pragma unroll
    for (int r = 0; r < QR; ++r) {
      b1[r] = b2[r] = b3[r] = INFINITY;
      s1[r] = s2[r] = 0;
      qx2[r] = pk2(q[r].x, q[r].x);
      qy2[r] = pk2(q[r].y, q[r].y);
      qz2[r] = pk2(q[r].z, q[r].z);
    }
    const uint32_t stage_s = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    for (int sub = wi; sub < nsub; sub += kRevWarps) {
      float tm[QR];
      if (staged) {
        // Candidates are pair-interleaved (pc_index): per 4 candidates four
        // broadcast LDS.128, six packed FFMA2 per query (each lane is d32()).
        const uint32_t sp = stage_s + static_cast<uint32_t>(sub * kSub) * 16u;
        float t0[QR], t1[QR];
#pragma unroll
        for (int r = 0; r < QR; ++r) t0[r] = t1[r] = INFINITY;
#pragma unroll
        for (int c = 0; c < kSub; c += 4) {
          const float4 A0 = lds128(sp + c * 16u), B0 = lds128(sp + (c + 1) * 16u);
          const float4 A1 = lds128(sp + (c + 2) * 16u), B1 = lds128(sp + (c + 3) * 16u);
#pragma unroll
          for (int r = 0; r < QR; ++r) {
            f32x2 d0 = ffma2(pk2(B0.x, B0.y), qz2[r], pk2(B0.z, B0.w));
            f32x2 d1 = ffma2(pk2(B1.x, B1.y), qz2[r], pk2(B1.z, B1.w));
            d0 = ffma2(pk2(A0.z, A0.w), qy2[r], d0);
            d1 = ffma2(pk2(A1.z, A1.w), qy2[r], d1);
            d0 = ffma2(pk2(A0.x, A0.y), qx2[r], d0);
            d1 = ffma2(pk2(A1.x, A1.y), qx2[r], d1);
            float l0, h0, l1, h1;
            up2(d0, l0, h0);
            up2(d1, l1, h1);
            t0[r] = fminf(t0[r], fminf(l0, h0));
            t1[r] = fminf(t1[r], fminf(l1, h1));
          }
        }
#pragma unroll
        for (int r = 0; r < QR; ++r) tm[r] = fminf(t0[r], t1[r]);
      } else {
#pragma unroll
        for (int r = 0; r < QR; ++r) {
          float t0 = INFINITY;
          for (int c = 0; c < kSub; ++c) t0 = fminf(t0, d32(q[r].x, q[r].y, q[r].z, pc_get(cand, sub * kSub + c)));
          tm[r] = t0;
        }
      }
#pragma unroll
      for (int r = 0; r < QR; ++r) {
        // Running top-3 of subtile minima (strict < keeps the earliest).
        const bool lt1 = tm[r] < b1[r], lt2 = tm[r] < b2[r];
        b3[r] = lt2 ? b2[r] : fminf(b3[r], tm[r]);
        s2[r] = lt1 ? s1[r] : (lt2 ? sub : s2[r]);
        b2[r] = lt1 ? b1[r] : (lt2 ? tm[r] : b2[r]);
        s1[r] = lt1 ? sub : s1[r];
        b1[r] = lt1 ? tm[r] : b1[r];
      }
    }
#pragma unroll
    for (int r = 0; r < QR; ++r) tops[wi * kRevWQ + lane + 32 * r] = RevTop{b1[r], b2[r], b3[r], s1[r], s2[r]};
    __syncthreads();
    if (tid >= w.nq) continue;
    // Epilogue: one thread per point merges the warps' top-3 lists and
    // certifies or decides the window.
    const int qlocal = w.q_first + tid;
    if (plan.fp64_mode) {
      push_refine(S, 1, w.owner, qlocal, 0, plan.iter);
      continue;
    }
    RevTop t = tops[tid];
#pragma unroll
    for (int k = 1; k < kRevWarps; ++k) {
      const RevTop o = tops[k * kRevWQ + tid];
      top3_insert(t.b1, t.s1, t.b2, t.s2, t.b3, o.b1, o.s1);
      top3_insert(t.b1, t.s1, t.b2, t.s2, t.b3, o.b2, o.s2);
      t.b3 = fminf(t.b3, o.b3);
    }
    const float4 qq = w.q[tid];
    int* slot = S.res_rev + static_cast<int64_t>(w.owner) * P.n_scene + qlocal;
    const float thr = __fadd_ru(t.b1, qq.w);
    bool ovf = t.b3 <= thr;
    int pos[kWinCap];
    int np = 0, pmin = -1;
    const int nscan = t.b2 <= thr ? 2 : 1;
    for (int sc = 0; sc < nscan; ++sc) {
      const int sid = sc == 0 ? t.s1 : t.s2;
      // Member bitmask in one pass, then the members in increasing position.
      unsigned mask = 0;
#pragma unroll 8
      for (int c = 0; c < kSub; ++c)
        mask |= (d32(qq.x, qq.y, qq.z, pc_get(cand, sid * kSub + c)) <= thr ? 1u : 0u) << c;
      while (mask) {
        const int c = __ffs(mask) - 1;
        mask &= mask - 1;
        const float d = d32(qq.x, qq.y, qq.z, pc_get(cand, sid * kSub + c));
        const int p = sid * kSub + c;
        if (np < kWinCap) pos[np] = p;
        ++np;
        if (d == t.b1 && (pmin < 0 || p < pmin)) pmin = p;
      }
    }
    ovf = ovf || np > kWinCap;
    if (ovf) {
      push_refine(S, 1, w.owner, qlocal, 1, plan.iter);
    } else if (np == 1) {
      *slot = pmin;  // certified
    } else {
      const NnGeom g = nn_geom(P, S, plan, 1, w.owner, qlocal);
      *slot = nn_decide(g, pos, np, false, S.stats);
    }
  }
}

// ---------------------------------------------------------------------------
// Forward / final filter on the tensor cores (ASICP_NN_TC=1).
//
// The distances of a (128 queries) x (256 candidates) tile are one K = 16
// tcgen05 MMA pair (kind::tf32, FP32 accumulators in TMEM) with a three-term
// TF32 split, hi*hi + hi*lo + lo*hi, which carries ~FP32 accuracy:
//   A row (query)     [qh 1 | qh 1 | ql 0 | 0]         (qh, ql: 3 floats each)
//   B row (candidate) [Bh nh | Bl nl | Bh 0 | 0]       (B = -2b, n = |b|^2)
// h = TF32-rounded (cvt.rna), l = the exact FP32 remainder; products of TF32
// operands are exact in FP32, so the error is the accumulation (<= 18 FP32
// roundings of partial sums bounded by S) plus the truncation of the l
// operands and the dropped l*l term: |d_tc - d| <= kTcErr * S with
// S = |b|^2 + 2 |q| |b| (measured <= 6.5 u S, tools/tc_nn_bench.cu; kTcErr =
// 64 u).
//
// nn_tc_kernel (one CTA per SM, warp-specialised): warps 0-1 gather the B
// tiles (candidate rows of the object's TF32 split, P.obj_tc, through the
// minibatch pool map) with cp.async into a 6-stage ring and build the A tile
// of each 128-query unit; warp 2 issues the MMAs into a double-buffered
// 2 x 256-column accumulator; warps 3-10 drain it (tcgen05.ld, one query per
// lane, two warps per lane quarter splitting the columns) into a running
// top-3 of 32-candidate subtile minima per query and split, written to
// S.tc_top.  nn_tc_window_kernel then certifies each (query, split) exactly
// as the FFMA2 filter's sub-chunk epilogue does, from the FP32 candidates:
// every candidate of the split's d32 window {d32 <= b1_32 + mg} has
// d_tc <= b1_tc + mg + 2 Et, so the subtiles s1 (and s2 when b2_tc is within
// that bound) hold the whole window and the split's d32 minimum; b3_tc within
// the bound sends the query to the full FP64 rescan.
// ---------------------------------------------------------------------------
constexpr int kTcM = 128, kTcN = 256, kTcK = 16;
constexpr int kTcStages = 6;
constexpr int kTcABytes = kTcM * kTcK * 4;
constexpr int kTcBBytes = kTcN * kTcK * 4;
constexpr int kTcProdWarps = 2, kTcEpiWarps = 8;  // + one MMA warp and one A-tile warp
constexpr int kTcMmaWarp = kTcProdWarps, kTcAWarp = kTcProdWarps + 1;
constexpr int kTcThreads = 32 * (kTcProdWarps + 2 + kTcEpiWarps);
constexpr int kTcBars = 2 * kTcStages + 2 + 2 + 2 + 2;  // full, empty, acc full/empty, A full/empty
// Dynamic shared memory: 1 KB alignment slack, A x 2, B ring, barriers; sized
// so that one CTA fits per SM (the kernel owns all 512 TMEM columns).
constexpr int kTcSmem = 1024 + 2 * kTcABytes + kTcStages * kTcBBytes + 256;
constexpr int kTcUnitsPerItem = kNnQB / kTcM;
constexpr float kTcErr = 3.8147e-06f;  // 64 u, u = 2^-24
constexpr uint32_t kTcIdesc =
    (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kTcN >> 3) << 17) | (static_cast<uint32_t>(kTcM >> 4) << 24);

// Float offset of (row r, k) in a K-major SWIZZLE_NONE tile: core matrices of
// 8 rows x 16 B, the next 4-float k chunk at +128 B (LBO), the next 8 rows at
// +512 B (SBO).
__host__ __device__ __forceinline__ int tc_off(int r, int k) {
  return (((r >> 3) * 4 + (k >> 2)) * 8 + (r & 7)) * 4 + (k & 3);
}
__device__ __forceinline__ uint64_t tc_sdesc(uint32_t saddr) {
  return ((saddr >> 4) & 0x3fffu) | (static_cast<uint64_t>(128 >> 4) << 16) | (static_cast<uint64_t>(512 >> 4) << 32) |
         (static_cast<uint64_t>(1) << 46);
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Wait with the thread suspended in hardware until the phase completes (the
// time hint only bounds a single try), so idle roles do not poll the issue
// slots the epilogue needs.
__device__ __forceinline__ void mbar_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(kTcIdesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async16_tc(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
#define TC_LD32(taddr, v)                                                                                        \
  asm volatile(                                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"  \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                              \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),  \
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),       \
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),      \
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                    \
      : "r"(taddr))

// Minimum of 32 accumulator values: a tree of 3-input mins (FMNMX3).
__device__ __forceinline__ float tc_min32(const uint32_t* x) {
  float m[11];
#pragma unroll
  for (int i = 0; i < 10; ++i)
    m[i] = fminf(fminf(__uint_as_float(x[3 * i]), __uint_as_float(x[3 * i + 1])), __uint_as_float(x[3 * i + 2]));
  m[10] = fminf(__uint_as_float(x[30]), __uint_as_float(x[31]));
  const float a0 = fminf(fminf(m[0], m[1]), m[2]), a1 = fminf(fminf(m[3], m[4]), m[5]);
  const float a2 = fminf(fminf(m[6], m[7]), m[8]), a3 = fminf(m[9], m[10]);
  return fminf(fminf(a0, a1), fminf(a2, a3));
}

// (v, s, mask) into a top-3 ordered by (value, subtile).
__device__ __forceinline__ void tc_top3_insert(float& b1, int& s1, unsigned& m1, float& b2, int& s2, unsigned& m2,
                                               float& b3, float v, int s, unsigned m) {
  if (v < b1 || (v == b1 && s < s1)) {
    b3 = b2;
    b2 = b1;
    s2 = s1;
    m2 = m1;
    b1 = v;
    s1 = s;
    m1 = m;
  } else if (v < b2 || (v == b2 && s < s2)) {
    b3 = b2;
    b2 = v;
    s2 = s;
    m2 = m;
  } else {
    b3 = fminf(b3, v);
  }
}

// The object's candidates as TF32 splits, 3 x 16 B per point:
// (Bh, nh), (Bl, nl), (Bh, 0) with B = -2b, n = |b|^2 from obj_cand4.
__global__ void obj_tc_kernel(const float4* cand4, int n, float4* tc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 v = cand4[i];
  const float hx = tf32_rna(v.x), hy = tf32_rna(v.y), hz = tf32_rna(v.z), hn = tf32_rna(v.w);
  tc[3 * i] = make_float4(hx, hy, hz, hn);
  tc[3 * i + 1] = make_float4(v.x - hx, v.y - hy, v.z - hz, v.w - hn);
  tc[3 * i + 2] = make_float4(hx, hy, hz, 0.0f);
}

void launch_obj_tc(const float4* cand4, int n, float4* tc, cudaStream_t st) {
  obj_tc_kernel<<<ceil_div(n, 256), 256, 0, st>>>(cand4, n, tc);
}

// The TC error bound of a query, Et = kTcErr (|b|^2 + 2 |q| |b|) over the
// object (B_obj = Bo), and its selection slack mg + 2 Et (see nn_tc_kernel),
// rounded up.
__device__ __forceinline__ float tc_et(float4 q, float Bo) {
  const float qa = __fsqrt_ru(__fmaf_ru(q.x, q.x, __fmaf_ru(q.y, q.y, __fmul_ru(q.z, q.z))));
  return __fmul_ru(kTcErr, __fmaf_ru(__fmul_ru(2.0f, qa), Bo, __fmul_ru(Bo, Bo)));
}
__device__ __forceinline__ float tc_slack(float4 q, float Bo) { return __fadd_ru(q.w, __fmul_ru(2.0f, tc_et(q, Bo))); }
// Candidates of a subtile whose TC value is within the slack of its minimum.
__device__ __forceinline__ unsigned tc_mask(const uint32_t* v, float lim) {
  unsigned m = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) m |= (__uint_as_float(v[i]) <= lim ? 1u : 0u) << i;
  return m;
}

struct TcUnit {
  int item, qt, nq;  // nq = 0: nothing to do
};
__device__ __forceinline__ TcUnit tc_unit(const DevState& S, int u) {
  TcUnit r;
  r.item = u / kTcUnitsPerItem;
  r.qt = u % kTcUnitsPerItem;
  r.nq = max(0, min(kTcM, S.items[0][r.item].nq - r.qt * kTcM));
  return r;
}

__global__ void __launch_bounds__(kTcThreads, 1) nn_tc_kernel(const __grid_constant__ DevProblem P,
                                                              const __grid_constant__ DevState S,
                                                              const __grid_constant__ NnPlan plan) {
  pdl_enter();
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  unsigned char* sm =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  float* sA = reinterpret_cast<float*>(sm);                   // 2 A tiles
  float* sB = reinterpret_cast<float*>(sm + 2 * kTcABytes);   // B ring
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 2 * kTcABytes + kTcStages * kTcBBytes);
  uint64_t *full = bars, *empty = bars + kTcStages, *accf = bars + 2 * kTcStages, *acce = accf + 2, *afull = acce + 2,
           *aempty = afull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kTcBars);
  __shared__ float xb[3][kTcM];
  __shared__ int xs[kTcM];
  __shared__ unsigned xm[2][kTcM];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Zero both A tiles and every B stage once: the k = 12..15 chunk is never
  // written again and must hold zeros (0 * garbage could be NaN).
  for (int i = tid; i < (2 * kTcABytes + kTcStages * kTcBBytes) / 16; i += kTcThreads)
    reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(full + s, 32 * kTcProdWarps);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf + b, 1);
      mbar_init(acce + b, 32 * kTcEpiWarps);
      mbar_init(afull + b, 32);
      mbar_init(aempty + b, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == kTcMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const int n_units = S.nn_dyn[1] * kTcUnitsPerItem;
  const uint32_t sA_s = smem_u32(sA), sB_s = smem_u32(sB);
  const float Bo = __double2float_ru(P.obj_meta[3]);

  if (warp < kTcProdWarps) {
    // B producer: the B tiles of every unit (cp.async gathers whose
    // completion arrives on the stage barrier).
    const int ptid = tid;
    int s = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const TcUnit U = tc_unit(S, u);
      if (U.nq == 0) continue;
      const NnItem w = S.items[0][U.item];
      const int* map = plan.pooled ? S.pool_idx + static_cast<int64_t>(w.owner) * P.n_obj_pad + w.c_base : nullptr;
      const int ntiles = ceil_div(w.nc, kTcN);
      // Candidate rows of this thread for tile t, loaded one tile ahead.
      constexpr int kPer = kTcN / (32 * kTcProdWarps);
      int rows[kPer], rows_next[kPer];
      auto load_rows = [&](int t, int* out) {
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int p = t * kTcN + ptid + i * 32 * kTcProdWarps;
          out[i] = p < w.nc ? (map ? __ldg(map + p) : w.c_base + p) : -1;
        }
      };
      load_rows(0, rows_next);
      for (int t = 0; t < ntiles; ++t) {
#pragma unroll
        for (int i = 0; i < kPer; ++i) rows[i] = rows_next[i];
        if (t + 1 < ntiles) load_rows(t + 1, rows_next);
        mbar_sleep(empty + s, ph ^ 1);
        const uint32_t bs = sB_s + static_cast<uint32_t>(s) * kTcBBytes;
        float* bg = sB + s * (kTcBBytes / 4);
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int cnd = ptid + i * 32 * kTcProdWarps;
          if (rows[i] >= 0) {
            const float4* src = P.obj_tc + 3 * static_cast<int64_t>(rows[i]);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
              cp_async16_tc(bs + static_cast<uint32_t>(tc_off(cnd, 4 * ch)) * 4u, src + ch);
          } else {
            // Padding rows: d = 1e30 (A's k = 3 entry is 1), never a minimum.
            *reinterpret_cast<float4*>(bg + tc_off(cnd, 0)) = make_float4(0.f, 0.f, 0.f, 1e30f);
            *reinterpret_cast<float4*>(bg + tc_off(cnd, 4)) = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(bg + tc_off(cnd, 8)) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        // The stage barrier counts this thread once its copies have landed
        // (no wait here); the MMA thread fences the generic-proxy writes.
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)) : "memory");
        if (++s == kTcStages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == kTcAWarp) {
    // A producer: the TF32 split of each unit's 128 queries, one unit ahead
    // of the MMAs (double-buffered), so unit boundaries do not stall the B
    // stream.
    int n = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const TcUnit U = tc_unit(S, u);
      if (U.nq == 0) continue;
      const float4* qs = S.items[0][U.item].q + U.qt * kTcM;
      float4 qv[kTcM / 32];
#pragma unroll
      for (int i = 0; i < kTcM / 32; ++i) {
        const int r = lane + 32 * i;
        qv[i] = r < U.nq ? qs[r] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const int ua = n & 1;
      mbar_sleep(aempty + ua, ((n >> 1) & 1) ^ 1);
      float* a = sA + ua * (kTcABytes / 4);
#pragma unroll
      for (int i = 0; i < kTcM / 32; ++i) {
        const int r = lane + 32 * i;
        const float4 q = qv[i];
        const float hx = tf32_rna(q.x), hy = tf32_rna(q.y), hz = tf32_rna(q.z);
        *reinterpret_cast<float4*>(a + tc_off(r, 0)) = make_float4(hx, hy, hz, 1.0f);
        *reinterpret_cast<float4*>(a + tc_off(r, 4)) = make_float4(hx, hy, hz, 1.0f);
        *reinterpret_cast<float4*>(a + tc_off(r, 8)) = make_float4(q.x - hx, q.y - hy, q.z - hz, 0.0f);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(afull + ua);
      ++n;
    }
  } else if (warp == kTcMmaWarp) {
    // MMA issuer (one lane).
    if (lane == 0) {
      int s = 0, b = 0;
      uint32_t ph = 0, aph = 0;
      int n = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const TcUnit U = tc_unit(S, u);
        if (U.nq == 0) continue;
        const int nc = S.items[0][U.item].nc;
        const int ua = n & 1;
        mbar_sleep(afull + ua, (n >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t as = sA_s + static_cast<uint32_t>(ua) * kTcABytes;
        const int ntiles = ceil_div(nc, kTcN);
        for (int t = 0; t < ntiles; ++t) {
          mbar_sleep(full + s, ph);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the gathered rows -> tensor core
          mbar_sleep(acce + b, aph ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t bs = sB_s + static_cast<uint32_t>(s) * kTcBBytes;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)  // k chunks 2kk, 2kk + 1: +256 B
            tc_mma(tmem + b * kTcN, tc_sdesc(as + kk * 256), tc_sdesc(bs + kk * 256), kk);
          tc_commit(empty + s);
          tc_commit(accf + b);
          if (++s == kTcStages) {
            s = 0;
            ph ^= 1;
          }
          if (++b == 2) {
            b = 0;
            aph ^= 1;
          }
        }
        tc_commit(aempty + ua);
        ++n;
      }
    }
  } else {
    // Epilogue: lane quarter (warp % 4), column half.
    const int ew = warp - kTcProdWarps - 2;
    const int quarter = warp & 3, half = ew >> 2;
    const int row = quarter * 32 + lane;
    int b = 0;
    uint32_t aph = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const TcUnit U = tc_unit(S, u);
      if (U.nq == 0) continue;
      const NnItem w = S.items[0][U.item];
      float b1 = INFINITY, b2 = INFINITY, b3 = INFINITY;
      int s1 = 0, s2 = 0;
      unsigned m1 = 0, m2 = 0;  // candidates of s1 / s2 within the slack of the subtile's minimum
      const float slack = row < U.nq ? tc_slack(w.q[U.qt * kTcM + row], Bo) : 0.0f;
      const int ntiles = ceil_div(w.nc, kTcN);
      for (int t = 0; t < ntiles; ++t) {
        mbar_sleep(accf + b, aph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t t0 = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + b * kTcN + half * (kTcN / 2);
#pragma unroll
        for (int sp = 0; sp < kTcN / 64; sp += 2) {
          uint32_t v0[32], v1[32];
          TC_LD32(t0 + sp * 32, v0);
          TC_LD32(t0 + sp * 32 + 32, v1);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const float tm0 = tc_min32(v0), tm1 = tc_min32(v1);
          const int sid = t * (kTcN / 32) + half * (kTcN / 64) + sp;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float tm = h ? tm1 : tm0;
            // Subtiles arrive in increasing order within the half: strict <
            // keeps the earliest (min/max network as in the FFMA2 filter).
            const bool lt1 = tm < b1, lt2 = tm < b2;
            b3 = fminf(b3, fmaxf(b2, tm));
            b2 = fminf(b2, fmaxf(b1, tm));
            b1 = fminf(b1, tm);
            s2 = lt1 ? s1 : (lt2 ? sid + h : s2);
            s1 = lt1 ? sid + h : s1;
            if (__any_sync(0xffffffffu, lt2)) {  // warp-uniform branch; rare after the first tiles
              const unsigned m = tc_mask(h ? v1 : v0, __fadd_ru(tm, slack));
              m2 = lt1 ? m1 : (lt2 ? m : m2);
              m1 = lt1 ? m : m1;
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(acce + b);
        if (++b == 2) {
          b = 0;
          aph ^= 1;
        }
      }
      // Merge the column halves (lexicographic (value, subtile) top-3).
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcEpiWarps));
      if (half == 1) {
        xb[0][row] = b1;
        xb[1][row] = b2;
        xb[2][row] = b3;
        xs[row] = s1 | (s2 << 16);
        xm[0][row] = m1;
        xm[1][row] = m2;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcEpiWarps));
      if (half == 0 && row < U.nq) {
        const int o12 = xs[row];
        tc_top3_insert(b1, s1, m1, b2, s2, m2, b3, xb[0][row], o12 & 0xffff, xm[0][row]);
        tc_top3_insert(b1, s1, m1, b2, s2, m2, b3, xb[1][row], o12 >> 16, xm[1][row]);
        b3 = fminf(b3, xb[2][row]);
        float4* o = S.tc_top + 2 * ((static_cast<int64_t>(w.slot) * w.nchunks + w.chunk) * kNnQB + U.qt * kTcM + row);
        o[0] = make_float4(b1, b2, b3, __int_as_float(s1 | (s2 << 16)));
        o[1] = make_float4(__uint_as_float(m1), __uint_as_float(m2), 0.0f, 0.0f);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == kTcMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Certification of the tensor-core top-3 (comment above nn_tc_kernel): one
// thread per (query, split).
__global__ void __launch_bounds__(kTcM) nn_tc_window_kernel(DevProblem P, DevState S, NnPlan plan) {
  pdl_enter();
  const int n_units = S.nn_dyn[1] * kTcUnitsPerItem;
  const float Bo = __double2float_ru(P.obj_meta[3]);
  for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
    const TcUnit U = tc_unit(S, u);
    if (U.nq == 0) continue;
    const NnItem w = S.items[0][U.item];
    if (threadIdx.x == 0) {
      const unsigned long long pairs = static_cast<unsigned long long>(U.nq) * w.nc;
      const unsigned long long nq0 = w.chunk == 0 ? U.nq : 0;
      atomicAdd(S.stats + 2, nq0);
      atomicAdd(S.stats + 4, pairs);
      atomicAdd(S.stats + 12, pairs);
      unsigned long long* is = S.iter_stats + 4 * plan.iter;
      atomicAdd(is, pairs);
      atomicAdd(is + 2, nq0);
    }
    const int r = threadIdx.x;
    if (r >= U.nq) continue;
    const int qi = U.qt * kTcM + r;
    const int qlocal = w.q_first + qi;
    const float4 q = w.q[qi];
    const float mg = q.w;
    const float4* tp = S.tc_top + 2 * ((static_cast<int64_t>(w.slot) * w.nchunks + w.chunk) * kNnQB + qi);
    const float4 T = tp[0];
    const float4 Tm = tp[1];
    const int s12 = __float_as_int(T.w);
    const float thr_sel = __fadd_ru(T.x, tc_slack(q, Bo));
    bool ovf = T.z <= thr_sel;
    const int nscan = T.y <= thr_sel ? 2 : 1;
    // The candidates of s1 (and s2) whose TC value is within the slack of
    // their subtile's minimum — a superset of the split's d32 window and of
    // its d32 minimum — in increasing position: their d32 values.
    const int sa = s12 & 0xffff, sb = s12 >> 16;
    const unsigned ma = __float_as_uint(Tm.x), mb = nscan == 2 ? __float_as_uint(Tm.y) : 0u;
    const bool a_first = nscan == 1 || sa < sb;
    int cpos[kWinCap + 1];
    float cd[kWinCap + 1];
    int nc = 0;
    float b1 = INFINITY;
    for (int sc = 0; sc < 2; ++sc) {
      const int sid = (sc == 0) == a_first ? sa : sb;
      unsigned m = (sc == 0) == a_first ? ma : mb;
      while (m) {
        const int c = __ffs(m) - 1;
        m &= m - 1;
        const float d = d32(q.x, q.y, q.z, pc_get(w.c, sid * kSub + c));
        b1 = fminf(b1, d);
        if (nc <= kWinCap) {
          cpos[nc] = w.c_base + sid * kSub + c;
          cd[nc] = d;
        }
        ++nc;
      }
    }
    if (nc > kWinCap) ovf = true;  // (not seen: masks hold one or two candidates)
    const float thr = __fadd_ru(b1, mg);
    int pos[kWinCap];
    float md[kWinCap];
    int np = 0, pmin = -1;
    for (int e = 0; e < min(nc, kWinCap); ++e) {
      if (cd[e] <= thr) {
        pos[np] = cpos[e];
        md[np] = cd[e];
        ++np;
        if (cd[e] == b1 && pmin < 0) pmin = cpos[e];
      }
    }
    ovf = ovf || np > kWinCap;
    if (w.nchunks == 1) {
      if (ovf) {
        push_refine(S, w.kind, w.owner, qlocal, 1, plan.iter);
      } else if (np == 1) {
        *nn_result_slot(P, S, w.kind, w.owner, qlocal) = pmin;  // certified
      } else {
        const NnGeom g = nn_geom(P, S, plan, w.kind, w.owner, qlocal);
        *nn_result_slot(P, S, w.kind, w.owner, qlocal) = nn_decide(g, pos, np, w.kind == 0 && !plan.pooled, S.stats);
      }
    } else {
      NnPartial pr;
      if (ovf) {
        // The split's minimum may lie in an unscanned subtile: a lower bound
        // keeps it in the merge's reach, and the unlisted window forces the
        // full rescan whenever it is.
        pr.b1 = __fsub_rd(T.x, tc_et(q, Bo));
        pr.pos = kAmbiguous | kNoBlock;
      } else if (np == 1) {
        pr.b1 = b1;
        pr.pos = pmin;
      } else {
        const int blk = win_alloc(S);
        if (blk >= 0) {
          S.amb_n[blk] = 0;
          for (int e = 0; e < np; ++e) win_push(S, blk, pos[e], md[e]);
        }
        pr.b1 = b1;
        pr.pos = kAmbiguous | (blk >= 0 ? blk : kNoBlock);
      }
      S.partials[(static_cast<int64_t>(w.slot) * w.nchunks + w.chunk) * kFwdQB + qi] = pr;
    }
  }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
void launch_nn_plan(const DevProblem& P, DevState& S, const NnPlan& plan, cudaStream_t st) {
  pdl_launch(nn_fill_kernel, dim3((P.J + kFillThreads - 1) / kFillThreads), dim3(kFillThreads), 0, st, P, S, plan);
}

int nn_smem_bytes() { return kNnSmem; }

void nn_set_attrs() {
  cudaFuncSetAttribute(nn_filter_kernel<kFwdQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNnSmem);
  cudaFuncSetAttribute(nn_rev_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRevSmem);
  cudaFuncSetAttribute(nn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_rev_blocks_per_sm, nn_rev_kernel, kRevThreads, kRevSmem);
  g_rev_blocks_per_sm = std::max(1, g_rev_blocks_per_sm);
}

int nn_blocks_per_sm() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, nn_filter_kernel<kFwdQ>, kNnThreads, kNnSmem);
  return n;
}

void launch_nn_rev(const DevProblem& P, DevState& S, const NnPlan& plan, int refine_grid, cudaStream_t st) {
  pdl_launch(nn_rev_kernel, dim3(refine_grid / 2 * g_rev_blocks_per_sm), dim3(kRevThreads), kRevSmem, st, P, S,
             plan);
}

int launch_nn(const DevProblem& P, DevState& S, const NnPlan& plan, int grid, int refine_grid, cudaStream_t st,
              cudaEvent_t ev_begin, cudaEvent_t ev_end, cudaEvent_t rev_done) {
  int n = 0;
  if (ev_begin) cudaEventRecord(ev_begin, st);
  if (plan.use_tc) {
    // Tensor-core filter (one CTA per SM) and its certification pass.
    pdl_launch(nn_tc_kernel, dim3(refine_grid / 2), dim3(kTcThreads), kTcSmem, st, P, S, plan);
    if (ev_end) cudaEventRecord(ev_end, st);
    pdl_launch(nn_tc_window_kernel, dim3(4 * refine_grid), dim3(kTcM), 0, st, P, S, plan);
    n += 2;
  } else {
    pdl_launch(nn_filter_kernel<kFwdQ>, dim3(grid), dim3(kNnThreads), kNnSmem, st, P, S, plan, 0);
    ++n;
    if (ev_end) cudaEventRecord(ev_end, st);
  }
  if (!rev_done && plan.kind == 0) {
    // refine_grid is two CTAs per SM; the reverse grid fills every SM.
    pdl_launch(nn_rev_kernel, dim3(refine_grid / 2 * g_rev_blocks_per_sm), dim3(kRevThreads), kRevSmem, st, P, S,
               plan);
    ++n;
  }
  if (plan.nchunks > 1) {
    dim3 mg((plan.max_ns + 127) / 128, P.J);
    pdl_launch(nn_merge_kernel, dim3(mg), dim3(128), 0, st, P, S, plan);
    ++n;
  }
  // A reverse match forked onto a side stream (launch_nn_rev) joins before
  // the refine, which serves both kinds' refine lists.
  if (rev_done) cudaStreamWaitEvent(st, rev_done, 0);
  pdl_launch(nn_refine_kernel, dim3(refine_grid), dim3(256), 0, st, P, S, plan);
  return n + 1;
}

}  // namespace asicp
