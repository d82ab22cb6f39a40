// Feasibility probe: the forward NN filter's distance evaluation on the
// tcgen05 tensor cores (kind::tf32, accumulators in TMEM) instead of packed
// FFMA2.  D[q][c] = |b_c|^2 - 2 q.b_c as a K = 16 GEMM with a three-term TF32
// split (hi*hi + hi*lo + lo*hi) so the products carry ~FP32 accuracy:
//
//   A row (query)     [qh.x qh.y qh.z 1 | qh.x qh.y qh.z 1 | ql.x ql.y ql.z 0 | 0 0 0 0]
//   B row (candidate) [Bh.x Bh.y Bh.z nh | Bl.x Bl.y Bl.z nl | Bh.x Bh.y Bh.z 0 | 0 0 0 0]
//   with B = -2 b, n = |b|^2, h = TF32-rounded, l = the exact FP32 remainder.
//
// One CTA per SM: warp 0 streams 256-candidate B tiles (bulk copies, 4-stage
// ring), warp 1 issues the MMAs (M128 N256, two K=8 steps) into a double-
// buffered TMEM accumulator, kEpiWarps warps drain it (tcgen05.ld 32x32b.x32,
// one query per lane, two warps per TMEM lane quarter splitting the columns)
// and keep the per-query minimum and its 32-candidate subtile.
// Reports (1) the TC error against the exact value of the same FP32 inputs and
// (2) pairs/s.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/tcb_bin tools/tc_nn_bench.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

constexpr int M = 128, N = 256, KF = 16;
constexpr int kStages = 4;
constexpr int kABytes = M * KF * 4;  // 8 KB
constexpr int kBBytes = N * KF * 4;  // 16 KB
constexpr int kEpiWarps = 8;         // two per TMEM lane quarter, each half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;

// Float offset of (row r, k) in a K-major SWIZZLE_NONE tile: core matrices of
// 8 rows x 16 bytes; LBO (next 4-float k chunk) = 128 B, SBO (next 8 rows) = 512 B.
__host__ __device__ inline int tile_off(int r, int k) { return (((r >> 3) * 4 + (k >> 2)) * 8 + (r & 7)) * 4 + (k & 3); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(smem_u32(b)), "r"(parity)
                 : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t sdesc(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3fff) | (uint64_t(128 >> 4) << 16) | (uint64_t(512 >> 4) << 32) | (uint64_t(1) << 46);
}
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define LD32(taddr, v)                                                                                          \
  asm volatile(                                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                             \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), \
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),      \
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),     \
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                   \
      : "r"(taddr))

// Minimum of 32 values as a tree of 3-input mins (FMNMX3), depth 4.
__device__ __forceinline__ float min32(const uint32_t* x) {
  float m[11];
#pragma unroll
  for (int i = 0; i < 10; ++i)
    m[i] = fminf(fminf(__uint_as_float(x[3 * i]), __uint_as_float(x[3 * i + 1])), __uint_as_float(x[3 * i + 2]));
  m[10] = fminf(__uint_as_float(x[30]), __uint_as_float(x[31]));
  const float a0 = fminf(fminf(m[0], m[1]), m[2]), a1 = fminf(fminf(m[3], m[4]), m[5]);
  const float a2 = fminf(fminf(m[6], m[7]), m[8]), a3 = fminf(m[9], m[10]);
  return fminf(fminf(a0, a1), fminf(a2, a3));
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_kernel(const float* __restrict__ A_all, const float* __restrict__ B_all, int n_qt, int n_ct, float* best_out,
              int* sub_out, float* dump) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  float* sA = reinterpret_cast<float*>(sm);
  float* sB = reinterpret_cast<float*>(sm + kABytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kABytes + kStages * kBBytes);
  uint64_t *full = bars, *empty = bars + kStages, *accf = bars + 2 * kStages, *acce = accf + 2, *afull = acce + 2,
           *aempty = afull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);
  __shared__ float hb[M];
  __shared__ int hs[M];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf + b, 1);
      mbar_init(acce + b, 32 * kEpiWarps);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0, it = 0;
      for (int qt = blockIdx.x; qt < n_qt; qt += gridDim.x, ++it) {
        mbar_wait(aempty, (it & 1) ^ 1);
        bulk_load(sA, A_all + static_cast<size_t>(qt) * M * KF, kABytes, afull);
        for (int ct = 0; ct < n_ct; ++ct) {
          mbar_wait(empty + s, ph ^ 1);
          bulk_load(sB + s * N * KF, B_all + static_cast<size_t>(ct) * N * KF, kBBytes, full + s);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int s = 0, b = 0;
      uint32_t ph = 0, aph = 0, it = 0;
      for (int qt = blockIdx.x; qt < n_qt; qt += gridDim.x, ++it) {
        mbar_wait(afull, it & 1);
        for (int ct = 0; ct < n_ct; ++ct) {
          mbar_wait(full + s, ph);
          mbar_wait(acce + b, aph ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const float* bt = sB + s * N * KF;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            mma_tf32(tmem + b * N, sdesc(sA + kk * 64), sdesc(bt + kk * 64), kk);  // +2 k chunks = +256 B
          mma_commit(empty + s);
          mma_commit(accf + b);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
          if (++b == 2) {
            b = 0;
            aph ^= 1;
          }
        }
        mma_commit(aempty);
      }
    }
  } else {
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    int b = 0;
    uint32_t aph = 0;
    for (int qt = blockIdx.x; qt < n_qt; qt += gridDim.x) {
      float best = INFINITY;
      int bsub = -1;
      for (int ct = 0; ct < n_ct; ++ct) {
        mbar_wait(accf + b, aph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t t0 = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + b * N + half * (N / 2);
#pragma unroll
        for (int sp = 0; sp < N / 64; sp += 2) {  // two 32-column subtiles per wait
          uint32_t v[32], w[32];
          LD32(t0 + sp * 32, v);
          LD32(t0 + sp * 32 + 32, w);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const float tv0 = min32(v), tv1 = min32(w);
          if (dump && qt == 0 && ct == 0)
            for (int i = 0; i < 32; ++i) {
              dump[row * N + half * (N / 2) + sp * 32 + i] = __uint_as_float(v[i]);
              dump[row * N + half * (N / 2) + (sp + 1) * 32 + i] = __uint_as_float(w[i]);
            }
          const int sub0 = ct * (N / 32) + half * (N / 64) + sp;
          if (tv0 < best) {
            best = tv0;
            bsub = sub0;
          }
          if (tv1 < best) {
            best = tv1;
            bsub = sub0 + 1;
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(acce + b);
        if (++b == 2) {
          b = 0;
          aph ^= 1;
        }
      }
      // The two halves' minima (ties: the lower subtile).
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
      if (half == 1) {
        hb[row] = best;
        hs[row] = bsub;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
      if (half == 0) {
        if (hb[row] < best || (hb[row] == best && hs[row] < bsub)) {
          best = hb[row];
          bsub = hs[row];
        }
        best_out[qt * M + row] = best;
        sub_out[qt * M + row] = bsub;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static float tf32_rna(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

int main(int argc, char** argv) {
  const int n_qt = argc > 1 ? atoi(argv[1]) : 148 * 4;
  const int n_ct = argc > 2 ? atoi(argv[2]) : 40;
  const int Q = n_qt * M, C = n_ct * N;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<float> U(-0.06f, 0.06f);
  std::vector<float> q(3 * Q), c(3 * C), nb(C);
  for (auto& v : q) v = U(rng);
  for (auto& v : c) v = U(rng);
  for (int i = 0; i < C; ++i) nb[i] = fmaf(c[3 * i], c[3 * i], fmaf(c[3 * i + 1], c[3 * i + 1], c[3 * i + 2] * c[3 * i + 2]));
  std::vector<float> A(static_cast<size_t>(Q) * KF, 0.f), B(static_cast<size_t>(C) * KF, 0.f);
  for (int i = 0; i < Q; ++i) {
    float* t = A.data() + static_cast<size_t>(i / M) * M * KF;
    const int r = i % M;
    for (int a = 0; a < 3; ++a) {
      const float h = tf32_rna(q[3 * i + a]), l = q[3 * i + a] - h;
      t[tile_off(r, a)] = h;
      t[tile_off(r, 4 + a)] = h;
      t[tile_off(r, 8 + a)] = l;
    }
    t[tile_off(r, 3)] = 1.f;
    t[tile_off(r, 7)] = 1.f;
  }
  for (int i = 0; i < C; ++i) {
    float* t = B.data() + static_cast<size_t>(i / N) * N * KF;
    const int r = i % N;
    for (int a = 0; a < 3; ++a) {
      const float x = -2.f * c[3 * i + a], h = tf32_rna(x), l = x - h;
      t[tile_off(r, a)] = h;
      t[tile_off(r, 4 + a)] = l;
      t[tile_off(r, 8 + a)] = h;
    }
    const float h = tf32_rna(nb[i]);
    t[tile_off(r, 3)] = h;
    t[tile_off(r, 7)] = nb[i] - h;
  }
  float *dA, *dB, *dbest, *ddump;
  int* dsub;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dbest, Q * 4);
  cudaMalloc(&dsub, Q * 4);
  cudaMalloc(&ddump, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = kABytes + kStages * kBBytes + 1024 + 256;
  cudaFuncSetAttribute(tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  tc_kernel<<<nsm, kThreads, smem>>>(dA, dB, n_qt, n_ct, dbest, dsub, ddump);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  // (1) accuracy of tile (qt 0, ct 0) against the exact value of the FP32 inputs
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), ddump, D.size() * 4, cudaMemcpyDeviceToHost);
  double max_rel = 0.0, max_abs = 0.0;
  for (int r = 0; r < M; ++r)
    for (int j = 0; j < N; ++j) {
      double ex = nb[j];
      double s = std::fabs(static_cast<double>(nb[j]));
      for (int a = 0; a < 3; ++a) {
        ex += -2.0 * c[3 * j + a] * static_cast<double>(q[3 * r + a]);
        s += std::fabs(2.0 * c[3 * j + a] * static_cast<double>(q[3 * r + a]));
      }
      const double err = std::fabs(D[r * N + j] - ex);
      max_abs = std::max(max_abs, err);
      max_rel = std::max(max_rel, err / s);
    }
  printf("TC vs exact (tile 0): max abs err %.3e, max err / sum|terms| %.3e (= %.2f x 2^-24)\n", max_abs, max_rel,
         max_rel / std::ldexp(1.0, -24));
  // (2) the per-query minimum against a CPU scan of a few queries
  std::vector<float> best(Q);
  std::vector<int> bsub(Q);
  cudaMemcpy(best.data(), dbest, Q * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(bsub.data(), dsub, Q * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < Q; i += 997) {
    double bv = INFINITY;
    int bs = -1;
    for (int j = 0; j < C; ++j) {
      double ex = nb[j];
      for (int a = 0; a < 3; ++a) ex += -2.0 * c[3 * j + a] * static_cast<double>(q[3 * i + a]);
      if (ex < bv) {
        bv = ex;
        bs = j / 32;
      }
    }
    if (std::fabs(best[i] - bv) > 1e-8 || (bsub[i] != bs && std::fabs(best[i] - bv) > 1e-9)) ++bad;
  }
  printf("per-query minimum: %d mismatches in %d sampled queries\n", bad, (Q + 996) / 997);
  // (3) throughput
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) tc_kernel<<<nsm, kThreads, smem>>>(dA, dB, n_qt, n_ct, dbest, dsub, nullptr);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int w = 0; w < reps; ++w) tc_kernel<<<nsm, kThreads, smem>>>(dA, dB, n_qt, n_ct, dbest, dsub, nullptr);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double pairs = static_cast<double>(Q) * C;
  printf("Q %d x C %d: %.3f ms per launch, %.2f T pairs/s (%.1f TFLOP/s tf32 at K=16)\n", Q, C, ms,
         pairs / ms / 1e9, pairs * 2 * KF / ms / 1e9);
  return 0;
}
