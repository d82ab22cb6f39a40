// Median-heuristic bandwidth for small and mid-size Stein populations
// (K <= kMedClusterK; larger ones: the grid-wide select in kernels.cu):
// h = max(median_{i<j} |t_i - t_j|^2 / log(K + 1), 1e-6) with the median the
// element nth_element places at M/2 (optim.cpp:133-144) — an exact order
// statistic, selected here on the FP64 bit patterns (non-negative doubles
// order like their bits).
//
// One CTA per population, everything in shared memory: the population's
// positions (K x 3 doubles), a 4096-bin histogram and a gather buffer.  Each
// pass recomputes the M = K(K-1)/2 keys from the staged positions (8 FP64
// operations), histograms the next 12 bits of the keys that match the
// selected prefix (warp-aggregated atomics: lanes holding the same digit add
// once) and picks the digit holding the target rank with a block scan.  As
// soon as the selected bucket holds at most kMedGather keys (two passes in
// practice: sign + exponent, then 12 mantissa bits), those keys are gathered,
// sorted (bitonic) and the rank is read off directly.  The row walk of the
// triangle is per thread (each thread strides by the block size).
#include "common.cuh"
#include "kernels.cuh"

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace cg = cooperative_groups;

namespace asicp {
namespace {

constexpr int kMedThreads = 1024;
constexpr int kMedBins = 4096;
// Gather once the bucket is this small: a bitonic sort of n keys costs
// ~log2(n)^2 / 2 block-wide phases, far more than one more radix pass when n
// is in the thousands (measured: 8192 -> ~80 % of the kernel).
constexpr int kMedGather = 1024;
constexpr int kMedSmem = kMedBigK * 3 * 8 + kMedBins * 4 + kMedGather * 8;

__device__ void block_bitonic_sort(unsigned long long* s, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = s[i], c = s[ixj];
          const bool asc = (i & k) == 0;
          if ((a > c) == asc) {
            s[i] = c;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kMedThreads) median_kernel(DevProblem P, DevState S) {
  pdl_enter();
  const int pop = blockIdx.x;
  if (P.pop_off[pop + 1] == P.pop_off[pop]) return;  // no local particle reads h
  const int b = P.gpop_off[pop], K = P.gpop_off[pop + 1] - b;
  if (K < 1) return;
  if (P.bandwidth_mode == 1) {
    if (threadIdx.x == 0) S.h[pop] = P.fixed_bandwidth;
    return;
  }
  if (K >= kMedBigK) return;  // grid-wide select (kernels.cu med_*_kernel)
  if (K < 2) {
    if (threadIdx.x == 0) S.h[pop] = 1.0;
    return;
  }
  extern __shared__ __align__(16) unsigned char med_smem[];
  double* tx = reinterpret_cast<double*>(med_smem);
  double* ty = tx + kMedBigK;
  double* tz = ty + kMedBigK;
  unsigned int* hist = reinterpret_cast<unsigned int*>(tz + kMedBigK);
  unsigned long long* gath = reinterpret_cast<unsigned long long*>(hist + kMedBins);
  __shared__ long long part[kMedThreads];
  __shared__ int s_digit, s_n;
  __shared__ long long s_below;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < K; i += blockDim.x) {
    const double* th = S.theta_all + 7 * static_cast<int64_t>(b + i);
    tx[i] = th[0];
    ty[i] = th[1];
    tz[i] = th[2];
  }
  const long long M = static_cast<long long>(K) * (K - 1) / 2;
  long long rank = M / 2;
  unsigned long long prefix = 0, mask = 0;
  // Visits every key once per call: f(valid, key) over 32 x 32 tiles of the
  // upper triangle (warp = one row i of the tile, lane = column j), i < j;
  // uniform trip count so warp collectives see full warps.
  auto for_keys = [&](auto&& f) {
    const int nb = (K + 31) / 32;
    const int ii = tid >> 5, jj = tid & 31;
    for (int bi = 0; bi < nb; ++bi) {
      const int i = bi * 32 + ii;
      for (int bj = bi; bj < nb; ++bj) {
        const int j = bj * 32 + jj;
        const bool valid = i < K && j < K && (bi < bj || ii < jj);
        unsigned long long key = 0;
        if (valid) {
          const double d2 = sqnorm(sub(V3{tx[i], ty[i], tz[i]}, V3{tx[j], ty[j], tz[j]}));
          key = static_cast<unsigned long long>(__double_as_longlong(d2));
        }
        f(valid, key);
      }
    }
  };
  const int shifts[6] = {52, 40, 28, 16, 4, 0}, widths[6] = {12, 12, 12, 12, 12, 4};
  for (int pass = 0; pass < 6; ++pass) {
    const int shift = shifts[pass];
    const unsigned int dmask = (1u << widths[pass]) - 1u;
    for (int i = tid; i < kMedBins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for_keys([&](bool valid, unsigned long long key) {
      const bool hit = valid && (key & mask) == prefix;
      const unsigned int digit = static_cast<unsigned int>(key >> shift) & dmask;
      const unsigned int active = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const unsigned int peers = __match_any_sync(active, digit);
        if (__ffs(peers) - 1 == lane) atomicAdd(&hist[digit], static_cast<unsigned int>(__popc(peers)));
      }
    });
    __syncthreads();
    // Digit holding `rank`: block scan of 4 bins per thread.
    long long mine = 0;
    for (int k = 0; k < kMedBins / kMedThreads; ++k) mine += hist[tid * (kMedBins / kMedThreads) + k];
    part[tid] = mine;
    __syncthreads();
    for (int off = 1; off < kMedThreads; off <<= 1) {
      const long long v = tid >= off ? part[tid - off] : 0;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    const long long before = tid ? part[tid - 1] : 0;
    if (rank >= before && rank < part[tid]) {
      long long acc = before;
      for (int k = 0; k < kMedBins / kMedThreads; ++k) {
        const int bin = tid * (kMedBins / kMedThreads) + k;
        if (rank < acc + hist[bin]) {
          s_digit = bin;
          s_below = acc;
          break;
        }
        acc += hist[bin];
      }
    }
    __syncthreads();
    const int digit = s_digit;
    const long long count = hist[digit];
    rank -= s_below;
    prefix |= static_cast<unsigned long long>(digit) << shift;
    mask |= static_cast<unsigned long long>(dmask) << shift;
    if (pass == 5) break;  // all 64 bits fixed: prefix is the key
    if (count <= kMedGather) {
      // Gather the bucket, sort it, read the rank.
      if (tid == 0) s_n = 0;
      __syncthreads();
      for_keys([&](bool valid, unsigned long long key) {
        const bool hit = valid && (key & mask) == prefix;
        const unsigned int bal = __ballot_sync(0xffffffffu, hit);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&s_n, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (hit) gath[base + __popc(bal & ((1u << lane) - 1u))] = key;
      });
      __syncthreads();
      int n2 = 2;
      while (n2 < count) n2 <<= 1;
      for (int e = static_cast<int>(count) + tid; e < n2; e += blockDim.x) gath[e] = ~0ull;
      __syncthreads();
      block_bitonic_sort(gath, n2);
      prefix = gath[rank];
      break;
    }
    __syncthreads();  // hist is reset by the next pass
  }
  if (tid == 0) {
    const double median = __longlong_as_double(static_cast<long long>(prefix));
    const double h = median / P.pop_logk1[pop];
    S.h[pop] = h < 1e-6 ? 1e-6 : h;  // std::max(h, 1e-6)
  }
}

// Mid-size populations (kMedBigK <= K <= kMedClusterK, e.g. cfg3 / cfg4's
// 1024 particles): the same select spread over a thread-block cluster of
// kMedCl CTAs.  Every CTA stages all K positions and owns every kMedCl-th
// 32 x 32 tile of the pair triangle; per pass each CTA histograms its keys
// into its own shared histogram, and after a cluster barrier every CTA sums
// the kMedCl histograms through distributed shared memory and picks the same
// digit (so no broadcast is needed).  The final bucket is gathered per CTA and
// merged by CTA 0, which sorts it and writes h.
constexpr int kMedCl = 8;
constexpr int kMedClSmem = kMedClusterK * 3 * 8 + kMedBins * 4 + kMedGather * 8;

__global__ void __cluster_dims__(kMedCl, 1, 1) __launch_bounds__(kMedThreads)
    median_cluster_kernel(DevProblem P, DevState S) {
  pdl_enter();
  const int pop = blockIdx.y;
  if (P.pop_off[pop + 1] == P.pop_off[pop]) return;  // uniform over the cluster
  const int b = P.gpop_off[pop], K = P.gpop_off[pop + 1] - b;
  if (P.bandwidth_mode == 1 || K < kMedBigK || K > kMedClusterK) return;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = static_cast<int>(cluster.block_rank());
  extern __shared__ __align__(16) unsigned char med_smem[];
  double* tx = reinterpret_cast<double*>(med_smem);
  double* ty = tx + kMedClusterK;
  double* tz = ty + kMedClusterK;
  unsigned int* hist = reinterpret_cast<unsigned int*>(tz + kMedClusterK);
  unsigned long long* gath = reinterpret_cast<unsigned long long*>(hist + kMedBins);
  __shared__ long long part[kMedThreads];
  __shared__ int s_digit, s_n;
  __shared__ long long s_below;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < K; i += blockDim.x) {
    const double* th = S.theta_all + 7 * static_cast<int64_t>(b + i);
    tx[i] = th[0];
    ty[i] = th[1];
    tz[i] = th[2];
  }
  const long long M = static_cast<long long>(K) * (K - 1) / 2;
  long long rank = M / 2;
  unsigned long long prefix = 0, mask = 0;
  // This CTA's keys: tiles (bi, bj >= bi) of the triangle in row-major order,
  // every kMedCl-th one; warp = row of the tile, lane = column.
  auto for_keys = [&](auto&& f) {
    const int nb = (K + 31) / 32;
    const int ii = tid >> 5, jj = tid & 31;
    // Tile crank, then every kMedCl-th: walk (bi, bj) forward kMedCl tiles.
    int bi = 0, bj = crank;
    for (;;) {
      // Normalise (bi, bj) to a tile of the triangle.
      while (bi < nb && bj >= nb) {
        bj = bi + 1 + (bj - nb);
        ++bi;
      }
      if (bi >= nb) break;
      const int i = bi * 32 + ii;
      const int j = bj * 32 + jj;
      const bool valid = i < K && j < K && (bi < bj || ii < jj);
      unsigned long long key = 0;
      if (valid) {
        const double d2 = sqnorm(sub(V3{tx[i], ty[i], tz[i]}, V3{tx[j], ty[j], tz[j]}));
        key = static_cast<unsigned long long>(__double_as_longlong(d2));
      }
      f(valid, key);
      bj += kMedCl;
    }
  };
  const int shifts[6] = {52, 40, 28, 16, 4, 0}, widths[6] = {12, 12, 12, 12, 12, 4};
  for (int pass = 0; pass < 6; ++pass) {
    const int shift = shifts[pass];
    const unsigned int dmask = (1u << widths[pass]) - 1u;
    for (int i = tid; i < kMedBins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for_keys([&](bool valid, unsigned long long key) {
      const bool hit = valid && (key & mask) == prefix;
      const unsigned int digit = static_cast<unsigned int>(key >> shift) & dmask;
      const unsigned int active = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const unsigned int peers = __match_any_sync(active, digit);
        if (__ffs(peers) - 1 == lane) atomicAdd(&hist[digit], static_cast<unsigned int>(__popc(peers)));
      }
    });
    cluster.sync();  // every CTA's histogram complete
    // Cluster-wide histogram (4 bins per thread) and the digit holding `rank`.
    constexpr int kPer = kMedBins / kMedThreads;
    unsigned int tot[kPer];
    long long mine = 0;
    for (int k = 0; k < kPer; ++k) {
      const int bin = tid * kPer + k;
      unsigned int s = 0;
      for (int r = 0; r < kMedCl; ++r) s += cluster.map_shared_rank(hist, r)[bin];
      tot[k] = s;
      mine += s;
    }
    part[tid] = mine;
    __syncthreads();
    for (int off = 1; off < kMedThreads; off <<= 1) {
      const long long v = tid >= off ? part[tid - off] : 0;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    const long long before = tid ? part[tid - 1] : 0;
    if (rank >= before && rank < part[tid]) {
      long long acc = before;
      for (int k = 0; k < kPer; ++k) {
        if (rank < acc + tot[k]) {
          s_digit = tid * kPer + k;
          s_below = acc;
          break;
        }
        acc += tot[k];
      }
    }
    __syncthreads();
    const int digit = s_digit;
    long long count = 0;
    for (int r = 0; r < kMedCl; ++r) count += cluster.map_shared_rank(hist, r)[digit];
    rank -= s_below;
    prefix |= static_cast<unsigned long long>(digit) << shift;
    mask |= static_cast<unsigned long long>(dmask) << shift;
    cluster.sync();  // every CTA done reading the histograms
    if (pass == 5) break;  // all 64 bits fixed: prefix is the key
    if (count <= kMedGather) {
      // Gather the bucket per CTA; CTA 0 merges, sorts and reads the rank.
      if (tid == 0) s_n = 0;
      __syncthreads();
      for_keys([&](bool valid, unsigned long long key) {
        const bool hit = valid && (key & mask) == prefix;
        const unsigned int bal = __ballot_sync(0xffffffffu, hit);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&s_n, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (hit) gath[base + __popc(bal & ((1u << lane) - 1u))] = key;
      });
      cluster.sync();  // every CTA's bucket part gathered
      if (crank == 0) {
        int off = s_n;
        for (int r = 1; r < kMedCl; ++r) {
          const int n = *cluster.map_shared_rank(&s_n, r);
          const unsigned long long* src = cluster.map_shared_rank(gath, r);
          for (int e = tid; e < n; e += blockDim.x) gath[off + e] = src[e];
          off += n;
        }
      }
      cluster.sync();  // CTA 0 done reading the other CTAs' shared memory
      if (crank == 0) {
        int n2 = 2;
        while (n2 < count) n2 <<= 1;
        for (int e = static_cast<int>(count) + tid; e < n2; e += blockDim.x) gath[e] = ~0ull;
        __syncthreads();
        block_bitonic_sort(gath, n2);
        prefix = gath[rank];
      }
      break;
    }
  }
  if (crank == 0 && tid == 0) {
    const double median = __longlong_as_double(static_cast<long long>(prefix));
    const double h = median / P.pop_logk1[pop];
    S.h[pop] = h < 1e-6 ? 1e-6 : h;  // std::max(h, 1e-6)
  }
}

}  // namespace

void median_set_attrs() {
  cudaFuncSetAttribute(median_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMedSmem);
  cudaFuncSetAttribute(median_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMedClSmem);
}

void launch_median_small(const DevProblem& P, DevState& S, cudaStream_t st) {
  pdl_launch(median_kernel, dim3(P.n_pop), dim3(kMedThreads), kMedSmem, st, P, S);
  if (P.med_mid) median_cluster_kernel<<<dim3(kMedCl, P.n_pop), kMedThreads, kMedClSmem, st>>>(P, S);
}

}  // namespace asicp
