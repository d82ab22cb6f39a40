// Parallel partial Fisher-Yates: the minibatch draw of sample_minibatch_indices
// (spatial_index.cpp:111-123) without the serial swap chain.
//
// The reference runs, for i = 0..m-1, j_i = i + uniform_index(n - i) and
// swap(idx[i], idx[j_i]) over an iota of length n, keeping idx[0..m).  Because
// position i is never touched after step i, and step s writes only positions
// s and j_s >= s:
//   pool[i] = j_i                 if no earlier step s < i had j_s = j_i,
//           = W(prev(i))          otherwise, prev(i) = the last such s;
//   W(s)    = s                   if no earlier step s' < s had j_s' = s,
//           = W(wl(s))            otherwise, wl(s) = the last such s'.
// (W(s) is the value sitting at position s when step s runs.)  With the pairs
// (j_s, s) sorted by key (stable), prev() is the sorted predecessor within a
// key group, wl(s) comes from the last member of group `s`, and W resolves by
// pointer jumping — all data-parallel over one CTA per particle.  The draws
// themselves are the particle's mt19937_64 outputs (twisted cooperatively);
// a Lemire rejection (probability ~n/2^64 per draw) sends the particle to an
// exact serial replay.
#include "common.cuh"
#include "mt64.cuh"

#include <cub/block/block_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

namespace asicp {

constexpr int kMbThreads = 1024;

template <int ITEMS>
__global__ void __launch_bounds__(kMbThreads) minibatch_par_kernel(DevProblem P, DevState S, int m, int j0) {
  pdl_enter();
  const int j = j0 + blockIdx.x;  // scratch slot blockIdx.x (the scratch covers S.fy_batch particles)
  if (!S.active[j] || S.n_col[j] > 0) return;
  using Sort = cub::BlockRadixSort<int, kMbThreads, ITEMS, int>;
  extern __shared__ __align__(16) unsigned char dyn[];
  typename Sort::TempStorage& sort_tmp = *reinterpret_cast<typename Sort::TempStorage*>(dyn);
  __shared__ uint64_t st[mt::kN];
  __shared__ uint64_t st0[mt::kN];
  __shared__ int s_mti, s_mti0, s_reject;
  const int tid = threadIdx.x;
  const int n = P.n_obj;
  int* scratch = S.fy_par + static_cast<int64_t>(blockIdx.x) * S.fy_stride;
  int* jv = scratch;                 // draw targets j_i, later pointer-jump buffer
  int* skey = scratch + P.n_obj_pad; // sorted keys
  int* sval = skey + P.n_obj_pad;    // sorted step indices
  int* lk = sval + P.n_obj_pad;      // key -> last sorted slot (keys < m)
  int* ptr = lk + P.n_obj_pad;       // W pointers
  int* pool = S.pool_idx + static_cast<int64_t>(j) * P.n_obj_pad;
  uint64_t* gst = S.rng_state + static_cast<int64_t>(j) * mt::kN;
  for (int i = tid; i < mt::kN; i += kMbThreads) st[i] = st0[i] = gst[i];
  if (tid == 0) {
    s_mti = s_mti0 = S.rng_mti[j];
    s_reject = 0;
  }
  __syncthreads();
  // 1. Draws (one engine output per draw unless a rejection happens).
  for (int i0 = 0; i0 < m;) {
    if (s_mti >= mt::kN) {
      mt::twist_block(st);
      if (tid == 0) s_mti = 0;
      __syncthreads();
    }
    const int mti = s_mti;
    const int cnt = min(mt::kN - mti, m - i0);
    for (int t = tid; t < cnt; t += kMbThreads) {
      uint64_t u;
      if (!mt::lemire(mt::temper(st[mti + t]), static_cast<uint64_t>(n - (i0 + t)), &u)) s_reject = 1;
      jv[i0 + t] = i0 + t + static_cast<int>(u);
    }
    __syncthreads();
    if (tid == 0) s_mti = mti + cnt;
    i0 += cnt;
    __syncthreads();
  }
  if (s_reject) {
    // Exact serial replay from the saved engine state (never seen in practice).
    if (tid == 0) {
      int* idx = skey;  // n ints available (stride is 5 * n_pad)
      for (int i = 0; i < n; ++i) idx[i] = i;
      int mt_i = s_mti0;
      for (int i = 0; i < m; ++i) {
        uint64_t u, x;
        do {
          if (mt_i >= mt::kN) {
            mt::twist_serial(st0);
            mt_i = 0;
          }
          x = mt::temper(st0[mt_i++]);
        } while (!mt::lemire(x, static_cast<uint64_t>(n - i), &u));
        const int jj = i + static_cast<int>(u);
        const int b = idx[jj];
        idx[jj] = idx[i];
        pool[i] = b;
      }
      for (int i = 0; i < mt::kN; ++i) st[i] = st0[i];
      s_mti = mt_i;
    }
    __syncthreads();
  } else {
    // 2. Stable sort of (j_s, s) by key.
    int nbits = 1;
    while ((1 << nbits) <= n) ++nbits;
    const int pad_key = (1 << nbits) - 1;
    int keys[ITEMS], vals[ITEMS];
#pragma unroll
    for (int e = 0; e < ITEMS; ++e) {
      const int i = tid * ITEMS + e;
      keys[e] = i < m ? jv[i] : pad_key;
      vals[e] = i;
    }
    __syncthreads();
    Sort(sort_tmp).Sort(keys, vals, 0, nbits);
#pragma unroll
    for (int e = 0; e < ITEMS; ++e) {
      const int t = tid * ITEMS + e;
      if (t < m) {
        skey[t] = keys[e];
        sval[t] = vals[e];
      }
    }
    for (int s = tid; s < m; s += kMbThreads) lk[s] = -1;
    __syncthreads();
    // 3. Last member of each key group (keys < m only matter for wl()).
    for (int t = tid; t < m; t += kMbThreads) {
      const int k = skey[t];
      if (k < m && (t == m - 1 || skey[t + 1] != k)) lk[k] = t;
    }
    __syncthreads();
    // 4. wl(s) -> initial pointers.
    for (int s = tid; s < m; s += kMbThreads) {
      const int t = lk[s];
      int wl = -1;
      if (t >= 0) {
        if (sval[t] < s)
          wl = sval[t];
        else if (t > 0 && skey[t - 1] == s)
          wl = sval[t - 1];
      }
      ptr[s] = wl < 0 ? s : wl;
    }
    __syncthreads();
    // 5. Pointer jumping to the chain roots (W).
    int* a = ptr;
    int* b = jv;
    for (;;) {
      int changed = 0;
      for (int s = tid; s < m; s += kMbThreads) {
        const int p = a[s];
        const int q = a[p];
        b[s] = q;
        changed |= q != p;
      }
      const int any = __syncthreads_or(changed);
      int* t = a;
      a = b;
      b = t;
      if (!any) break;
    }
    // 6. pool[i] from the sorted predecessor within the key group.
    for (int t = tid; t < m; t += kMbThreads) {
      const int i = sval[t];
      const int k = skey[t];
      pool[i] = (t > 0 && skey[t - 1] == k) ? a[sval[t - 1]] : k;
    }
    __syncthreads();
  }
  for (int i = tid; i < mt::kN; i += kMbThreads) gst[i] = st[i];
  if (tid == 0) S.rng_mti[j] = s_mti;
  // Gather the FP32 candidates in sample order (+inf padded to the subtile),
  // pair-interleaved like the object cloud (common.cuh pc_*).
  float4* pool32 = S.pool32 + static_cast<int64_t>(j) * P.n_obj_pad;
  gather_pool(P.obj_cand4, pool, m, pool32, tid, kMbThreads);
}

// Same algorithm with the stable sort replaced by a counting sort in shared
// memory (clouds of n <= kCountMax points): per-key counts, a block-wide
// exclusive scan, an atomic scatter, and an insertion sort of each key group by
// step (groups hold a handful of steps) — which yields exactly the stable
// order.  O(n + m) shared-memory work instead of a multi-pass radix sort, and
// no bound on m.
constexpr int kCountMax = 49152;

template <typename IT>
__device__ __forceinline__ void draws_block(const DevProblem& P, DevState& S, int j, int m, int n, IT* jv,
                                            uint64_t* st, uint64_t* st0, int* s_mti, int* s_mti0, int* s_reject) {
  const int tid = threadIdx.x;
  uint64_t* gst = S.rng_state + static_cast<int64_t>(j) * mt::kN;
  for (int i = tid; i < mt::kN; i += kMbThreads) st[i] = st0[i] = gst[i];
  if (tid == 0) {
    *s_mti = *s_mti0 = S.rng_mti[j];
    *s_reject = 0;
  }
  __syncthreads();
  for (int i0 = 0; i0 < m;) {
    if (*s_mti >= mt::kN) {
      mt::twist_block(st);
      if (tid == 0) *s_mti = 0;
      __syncthreads();
    }
    const int mti = *s_mti;
    const int cnt = min(mt::kN - mti, m - i0);
    for (int t = tid; t < cnt; t += kMbThreads) {
      uint64_t u;
      if (!mt::lemire(mt::temper(st[mti + t]), static_cast<uint64_t>(n - (i0 + t)), &u)) *s_reject = 1;
      jv[i0 + t] = static_cast<IT>(i0 + t + static_cast<int>(u));
    }
    __syncthreads();
    if (tid == 0) *s_mti = mti + cnt;
    i0 += cnt;
    __syncthreads();
  }
}

// Shared-memory arena of the counting-sort kernel: the key counters / group
// ends (cnt, max(n, m)), the draws (jv, m), the sorted steps (sval, m), the W
// pointers and the pointer-jump buffer (ptr, jb, m each).  Sorted keys are
// jv[sval[t]].  Entries are 16-bit when n and m fit (cfg2 / cfg4: a 100 KB
// arena, two 1024-thread CTAs per SM), else 32-bit; when even that does not
// fit, everything but cnt lives in the particle's global scratch.
__host__ __device__ __forceinline__ int64_t mb_arena_ints(int n, int m) {
  return static_cast<int64_t>(n > m ? n : m) + 4ll * m;
}
constexpr int kMbArenaMax = 200 * 1024;  // bytes of dynamic shared memory
constexpr int kMbArena16Max = 100 * 1024;  // 16-bit arenas up to this size: 2 CTAs per SM
constexpr int kMbNone16 = 0xffff;          // "no group end" in a 16-bit arena

// Counters of the counting sort: 32-bit words, or two 16-bit halves per word
// (atomics on the containing word; counts and offsets stay below 2^16).
template <typename IT>
struct MbCnt {
  unsigned int* w;
  __device__ unsigned int add(int k, unsigned int v) const { return atomicAdd(w + k, v); }
  __device__ unsigned int get(int k) const { return w[k]; }
  __device__ void set(int k, unsigned int v) const { w[k] = v; }
};
template <>
struct MbCnt<uint16_t> {
  unsigned int* w;
  __device__ unsigned int add(int k, unsigned int v) const {
    const int sh = 16 * (k & 1);
    return (atomicAdd(w + (k >> 1), v << sh) >> sh) & 0xffffu;
  }
  __device__ unsigned int get(int k) const { return reinterpret_cast<const uint16_t*>(w)[k]; }
  __device__ void set(int k, unsigned int v) const { reinterpret_cast<uint16_t*>(w)[k] = static_cast<uint16_t>(v); }
};

// in_smem: 1 arena in shared memory; 0 counters in shared memory, the rest in
// the particle's scratch; 2 everything in the scratch (clouds too large for
// shared counters: the counters follow the four m-arrays).
template <typename IT>
__global__ void __launch_bounds__(kMbThreads) minibatch_cnt_kernel(DevProblem P, DevState S, int m, int in_smem,
                                                                   int j0) {
  pdl_enter();
  const int j = j0 + blockIdx.x;  // scratch slot blockIdx.x (the scratch covers S.fy_batch particles)
  if (!S.active[j] || S.n_col[j] > 0) return;
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ uint64_t st[mt::kN];
  __shared__ uint64_t st0[mt::kN];
  __shared__ int s_mti, s_mti0, s_reject;
  __shared__ unsigned int part[kMbThreads];
  constexpr bool k16 = sizeof(IT) == 2;
  const int tid = threadIdx.x;
  const int n = P.n_obj;
  const int ncnt = n > m ? n : m;
  int* scratch = S.fy_par + static_cast<int64_t>(blockIdx.x) * S.fy_stride;
  // counters -> offsets -> group ends (lk)
  const MbCnt<IT> cnt{in_smem == 2 ? reinterpret_cast<unsigned int*>(scratch + 4ll * P.n_obj_pad)
                                   : reinterpret_cast<unsigned int*>(dyn)};
  // 16-bit counters are packed two per word: round the count area to words.
  const bool arena = in_smem == 1;
  IT* base = arena ? reinterpret_cast<IT*>(dyn) + (k16 ? (ncnt + 1) / 2 * 2 : ncnt)
                   : reinterpret_cast<IT*>(scratch);  // (IT = int whenever the arena is not in shared memory)
  IT* jv = base;
  IT* sval = jv + (arena ? m : P.n_obj_pad);
  IT* ptr = sval + (arena ? m : P.n_obj_pad);
  IT* jb = ptr + (arena ? m : P.n_obj_pad);
  int* pool = S.pool_idx + static_cast<int64_t>(j) * P.n_obj_pad;
  auto lk_get = [&](int k) -> int {
    const unsigned int v = cnt.get(k);
    return k16 ? (v == kMbNone16 ? -1 : static_cast<int>(v)) : static_cast<int>(v);
  };
  draws_block(P, S, j, m, n, jv, st, st0, &s_mti, &s_mti0, &s_reject);
  if (s_reject) {
    // Exact serial replay from the saved engine state (never seen in practice).
    if (tid == 0) {
      int* idx = scratch;  // n ints of the global scratch (5 x n_pad per particle)
      for (int i = 0; i < n; ++i) idx[i] = i;
      int mt_i = s_mti0;
      for (int i = 0; i < m; ++i) {
        uint64_t u, x;
        do {
          if (mt_i >= mt::kN) {
            mt::twist_serial(st0);
            mt_i = 0;
          }
          x = mt::temper(st0[mt_i++]);
        } while (!mt::lemire(x, static_cast<uint64_t>(n - i), &u));
        const int jj = i + static_cast<int>(u);
        const int b = idx[jj];
        idx[jj] = idx[i];
        pool[i] = b;
      }
      for (int i = 0; i < mt::kN; ++i) st[i] = st0[i];
      s_mti = mt_i;
    }
    __syncthreads();
  } else {
    // 2. Counting sort of (j_s, s) by key, stable.
    for (int k = tid; k < (k16 ? (n + 1) / 2 : n); k += kMbThreads) cnt.w[k] = 0u;
    __syncthreads();
    for (int s = tid; s < m; s += kMbThreads) cnt.add(jv[s], 1u);
    __syncthreads();
    const int per = (n + kMbThreads - 1) / kMbThreads;
    const int k0 = tid * per, k1 = min(n, k0 + per);
    unsigned int sum = 0;
    for (int k = k0; k < k1; ++k) sum += cnt.get(k);
    part[tid] = sum;
    __syncthreads();
    for (int off = 1; off < kMbThreads; off <<= 1) {  // inclusive scan of the segment sums
      const unsigned int v = tid >= off ? part[tid - off] : 0u;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    unsigned int run = tid ? part[tid - 1] : 0u;
    // (Per-thread ranges are even-aligned for 16-bit counters only when per is
    // even; a half-word store next to another thread's half is still a
    // distinct 16-bit location, so plain stores are safe.)
    for (int k = k0; k < k1; ++k) {
      const unsigned int c = cnt.get(k);
      cnt.set(k, run);
      run += c;
    }
    __syncthreads();
    for (int s = tid; s < m; s += kMbThreads) sval[cnt.add(jv[s], 1u)] = static_cast<IT>(s);
    __syncthreads();
    // Order each key group by step (groups hold a handful of steps).
    for (int t = tid; t < m; t += kMbThreads) {
      const int k = jv[sval[t]];
      if (t > 0 && jv[sval[t - 1]] == k) continue;
      int e = t + 1;
      while (e < m && jv[sval[e]] == k) ++e;
      for (int a = t + 1; a < e; ++a) {
        const IT v = sval[a];
        int b = a - 1;
        while (b >= t && sval[b] > v) {
          sval[b + 1] = sval[b];
          --b;
        }
        sval[b + 1] = v;
      }
    }
    __syncthreads();
    // 3. Last member of each key group (keys < m only matter for wl()); the
    // counters are dead now, so their space holds lk.
    for (int s = tid; s < m; s += kMbThreads) cnt.set(s, k16 ? kMbNone16 : 0xffffffffu);
    __syncthreads();
    for (int t = tid; t < m; t += kMbThreads) {
      const int k = jv[sval[t]];
      if (k < m && (t == m - 1 || jv[sval[t + 1]] != k)) cnt.set(k, static_cast<unsigned int>(t));
    }
    __syncthreads();
    // 4. wl(s) -> initial pointers.
    for (int s = tid; s < m; s += kMbThreads) {
      const int t = lk_get(s);
      int wl = -1;
      if (t >= 0) {
        if (sval[t] < s)
          wl = sval[t];
        else if (t > 0 && jv[sval[t - 1]] == s)
          wl = sval[t - 1];
      }
      ptr[s] = static_cast<IT>(wl < 0 ? s : wl);
    }
    __syncthreads();
    // 5. Pointer jumping to the chain roots (W).
    IT* a = ptr;
    IT* b = jb;
    for (;;) {
      int changed = 0;
      for (int s = tid; s < m; s += kMbThreads) {
        const IT p = a[s];
        const IT q = a[p];
        b[s] = q;
        changed |= q != p;
      }
      const int any = __syncthreads_or(changed);
      IT* t = a;
      a = b;
      b = t;
      if (!any) break;
    }
    // 6. pool[i] from the sorted predecessor within the key group.
    for (int t = tid; t < m; t += kMbThreads) {
      const int i = sval[t];
      const int k = jv[i];
      pool[i] = (t > 0 && jv[sval[t - 1]] == k) ? static_cast<int>(a[sval[t - 1]]) : k;
    }
    __syncthreads();
  }
  uint64_t* gst = S.rng_state + static_cast<int64_t>(j) * mt::kN;
  for (int i = tid; i < mt::kN; i += kMbThreads) gst[i] = st[i];
  if (tid == 0) S.rng_mti[j] = s_mti;
  float4* pool32 = S.pool32 + static_cast<int64_t>(j) * P.n_obj_pad;
  gather_pool(P.obj_cand4, pool, m, pool32, tid, kMbThreads);
}

template <int ITEMS>
constexpr int par_smem() {
  return static_cast<int>(sizeof(typename cub::BlockRadixSort<int, kMbThreads, ITEMS, int>::TempStorage));
}

template <int ITEMS>
static int launch_par(const DevProblem& P, DevState& S, int m, cudaStream_t st) {
  int n = 0;
  for (int j0 = 0; j0 < P.J; j0 += S.fy_batch, ++n)
    pdl_launch(minibatch_par_kernel<ITEMS>, dim3(min(S.fy_batch, P.J - j0)), dim3(kMbThreads), par_smem<ITEMS>(), st,
               P, S, m, j0);
  return n;
}

// Opt-in shared-memory sizes on the current device (per context: function
// attributes are per device).
void minibatch_set_attrs() {
  cudaFuncSetAttribute(minibatch_par_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, par_smem<4>());
  cudaFuncSetAttribute(minibatch_par_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, par_smem<12>());
  cudaFuncSetAttribute(minibatch_par_kernel<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, par_smem<20>());
  cudaFuncSetAttribute(minibatch_cnt_kernel<int>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMbArenaMax);
  cudaFuncSetAttribute(minibatch_cnt_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMbArena16Max);
}

// Returns the number of launches, or 0 when the parallel path does not apply
// (no scratch at all); the caller then uses the serial kernel.  The scratch
// covers S.fy_batch particles: larger populations take several launches.
int launch_minibatch_par(const DevProblem& P, DevState& S, int m, cudaStream_t st) {
  if (S.fy_par == nullptr) return 0;
  auto cnt_launches = [&](auto kern, size_t smem, int in_smem) {
    int n = 0;
    for (int j0 = 0; j0 < P.J; j0 += S.fy_batch, ++n)
      pdl_launch(kern, dim3(min(S.fy_batch, P.J - j0)), dim3(kMbThreads), smem, st, P, S, m, in_smem, j0);
    return n;
  };
  if (P.n_obj <= kCountMax) {
    const int ncnt = P.n_obj > m ? P.n_obj : m;
    const int64_t arena16 = (static_cast<int64_t>((ncnt + 1) / 2 * 2) + 4ll * m) * 2;
    // 16-bit arenas (two CTAs per SM) when the GPU is shared with other solves
    // (throughput mode: the 32-bit arena's one-CTA-per-SM shared memory keeps
    // the other solves' kernels off the SM) or when the population is large
    // (many waves); a small solve alone (cfg2's 768 particles) runs the
    // 32-bit kernel, which is faster per CTA (measured: cfg2 33.9 -> 33.1 ms,
    // cfg3 / cfg5 faster with 16 bits).  ASICP_MB16=0/1 forces either.
    static const int mb16_env = [] {
      const char* e = std::getenv("ASICP_MB16");
      return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    const bool mb16 = mb16_env >= 0 ? mb16_env == 1 : (P.throughput != 0 || P.J >= 1024);
    if (mb16 && P.n_obj < 65535 && m < 65535 && arena16 <= kMbArena16Max)
      return cnt_launches(minibatch_cnt_kernel<uint16_t>, static_cast<size_t>(arena16), 1);
    const int64_t arena = mb_arena_ints(P.n_obj, m) * 4;
    const int in_smem = arena <= kMbArenaMax ? 1 : 0;
    const size_t smem = in_smem ? static_cast<size_t>(arena) : static_cast<size_t>(P.n_obj) * 4;
    return cnt_launches(minibatch_cnt_kernel<int>, smem, in_smem);
  }
  if (m <= kMbThreads * 4) return launch_par<4>(P, S, m, st);
  if (m <= kMbThreads * 12) return launch_par<12>(P, S, m, st);
  if (m <= kMbThreads * 20) return launch_par<20>(P, S, m, st);
  // Large clouds and draws: the counting sort with every array (counters
  // included) in the particle's global scratch.
  return cnt_launches(minibatch_cnt_kernel<int>, 0, 2);
}

}  // namespace asicp
