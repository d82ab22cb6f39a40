// Device helpers shared by kernels.cu and nn.cu.
#pragma once

#include "dmath.cuh"
#include "kernels.cuh"

#include <cstdint>

namespace asicp {

// Programmatic dependent launch (PDL).  Every kernel of the solve begins with
// pdl_enter(): it lets the next kernel of the stream launch right away (its
// CTAs are placed as this grid's CTAs retire and then wait in their own
// pdl_enter), then waits until the previous kernel has completed and its
// writes are visible.  Launch-to-launch gaps of the ~1,200-node solve graph
// shrink to the wait.  A kernel launched without the attribute passes through.
__device__ __forceinline__ void pdl_enter() {
#ifdef ASICP_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... K, typename... A>
inline void pdl_launch(void (*kern)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<K>(args)...);
}

constexpr int kSub = 32;  // NN candidates per subtile (the unit of window tracking)

__device__ __forceinline__ const double* th_of(const double* theta, int j) { return theta + 7 * j; }

__device__ __forceinline__ V3 load3(const double* p, int64_t i) { return V3{p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }

__host__ __device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int round_up(int a, int b) { return ceil_div(a, b) * b; }

// Rigorous bound on the FP32 expansion-form distance error:
// with a = query - centre, b = candidate - centre, A = |a|, B >= max |b|,
//   |d32 - (|b|^2 - 2 a.b)| <= E = 1.01 u (6 B^2 + 10 A B) + 2^-50 (A + B)^2,
// u = 2^-24 (the 2^-50 term covers the reference's own FP64 rounding).  Two
// candidates whose FP32 values differ by more than 2E are ordered correctly,
// so the window [b1, b1 + 2E] contains the reference's answer.
__device__ __forceinline__ float nn_margin(double A, double B) {
  const double u = 5.9604644775390625e-08;
  const double e32 = 1.01 * u * (6.0 * B * B + 10.0 * A * B);
  const double e64 = 8.881784197001252e-16 * (A + B) * (A + B);
  return __double2float_ru(2.0 * (e32 + e64));
}

// The same bound evaluated in FP32 with upward rounding (A, B upper bounds).
__device__ __forceinline__ float nn_margin32(float A, float B) {
  const float e32 = __fmul_ru(6.0206e-08f /* 1.01 u, rounded up */,
                              __fadd_ru(__fmul_ru(6.0f, __fmul_ru(B, B)), __fmul_ru(10.0f, __fmul_ru(A, B))));
  const float s = __fadd_ru(A, B);
  const float e64 = __fmul_ru(8.881784197001252e-16f, __fmul_ru(s, s));
  return __fmul_ru(2.0f, __fadd_ru(e32, e64));
}

// Forward NN candidates (the object cloud and the minibatch pools) are stored
// pair-interleaved: candidates 2p and 2p + 1 occupy two float4s,
// (x0, x1, y0, y1) and (z0, z1, w0, w1), so one LDS.128 yields ready-made
// register pairs for the packed FFMA2 of the NN filter.  16 B per candidate
// as before; splits and tiles start at even candidates.
__host__ __device__ __forceinline__ int64_t pc_index(int64_t c) { return (c >> 1) * 8 + (c & 1); }
__device__ __forceinline__ float4 pc_get(const float4* base, int64_t c) {
  const float* f = reinterpret_cast<const float*>(base) + pc_index(c);
  return make_float4(f[0], f[2], f[4], f[6]);
}
__device__ __forceinline__ void pc_put(float4* base, int64_t c, float4 v) {
  float* f = reinterpret_cast<float*>(base) + pc_index(c);
  f[0] = v.x;
  f[2] = v.y;
  f[4] = v.z;
  f[6] = v.w;
}

// Minibatch pool gather: pool32 = candidates pool[0..m) in sample order,
// pair-interleaved (pc_index) and +inf padded to the subtile.  A thread writes
// one candidate pair: two 16-byte loads from the plain copy, two 16-byte
// stores (the per-float pc_get / pc_put took four of each per candidate).
__device__ __forceinline__ void gather_pool(const float4* cand4, const int* pool, int m, float4* pool32, int tid,
                                            int nt) {
  const int mp = round_up(m, kSub);
  const float4 pad = make_float4(0.0f, 0.0f, 0.0f, INFINITY);
  for (int i2 = 2 * tid; i2 < mp; i2 += 2 * nt) {
    const float4 a = i2 < m ? cand4[pool[i2]] : pad;
    const float4 b = i2 + 1 < m ? cand4[pool[i2 + 1]] : pad;
    pool32[i2] = make_float4(a.x, b.x, a.y, b.y);
    pool32[i2 + 1] = make_float4(a.z, b.z, a.w, b.w);
  }
}

// True contact-surface size of particle j (surface rows are padded to kSub).
__device__ __forceinline__ int surf_count(const DevProblem& P, int j) {
  const int pre = P.part_pre[j];
  return P.pre_surf_off[pre + 1] - P.pre_surf_off[pre];
}

}  // namespace asicp
