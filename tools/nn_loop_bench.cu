// Ceiling of the NN filter's inner loop (diagnostic): the packed-FFMA2 hot
// loop of nn_filter_kernel (nn.cu) over a shared-memory tile, alone and with
// the per-subtile top-3 update, at several CTAs per SM.  Prints pairs/clk/SM
// and the FMA-pipe fraction (3 FMA per pair, 128 FMA/clk/SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nn_loop_bench tools/nn_loop_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

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

constexpr int kSub = 32, kCand = 2048;

// MODE 0: hot loop only, 1: + top-3 per subtile, 2: + top-3 with the queries
// held as pre-packed register pairs (no .F32 broadcast operand), 3: scalar
// FFMA form + top-3.  Queries come from global memory (no constant folding).
template <int MODE, int Q = 8, int MINB = 4, int UNR = 2, int TRACK = 32, bool NET = false>
__global__ void __launch_bounds__(128, MINB) loop_kernel(const float4* cand, const float4* qin, float* out, int reps) {
  __shared__ float4 tile[kCand];
  for (int i = threadIdx.x; i < kCand; i += blockDim.x) tile[i] = cand[i];
  __syncthreads();
  float qx[Q], qy[Q], qz[Q];
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    const float4 q = qin[(blockIdx.x * 128 + threadIdx.x) * Q + k];
    qx[k] = q.x;
    qy[k] = q.y;
    qz[k] = q.z;
  }
  f32x2 px[Q], py[Q], pz[Q];
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    px[k] = pk2(qx[k], qx[k]);
    py[k] = pk2(qy[k], qy[k]);
    pz[k] = pk2(qz[k], qz[k]);
  }
  float b1[Q], b2[Q], b3[Q];
  int s12[Q];
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    b1[k] = b2[k] = b3[k] = INFINITY;
    s12[k] = 0;
  }
  for (int r = 0; r < reps; ++r) {
    for (int sub = 0; sub < kCand / TRACK; ++sub) {
      const float4* sp = tile + sub * TRACK;
      float tm[Q];
#pragma unroll
      for (int k = 0; k < Q; ++k) tm[k] = INFINITY;
      if (MODE == 3) {
#pragma unroll 4
        for (int c = 0; c < kSub; c += 2) {
          const float4 A = sp[c], B = sp[c + 1];
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            const float d0 = __fmaf_rn(qx[k], A.x, __fmaf_rn(qy[k], A.z, __fmaf_rn(qz[k], B.x, B.z)));
            const float d1 = __fmaf_rn(qx[k], A.y, __fmaf_rn(qy[k], A.w, __fmaf_rn(qz[k], B.y, B.w)));
            tm[k] = fminf(tm[k], fminf(d0, d1));
          }
        }
      } else {
#pragma unroll UNR
      for (int c = 0; c < TRACK; c += 4) {
        const float4 a0 = sp[c], c0 = sp[c + 1];
        const float4 a1 = sp[c + 2], c1 = sp[c + 3];
        const f32x2 x0 = pk2(a0.x, a0.y), y0 = pk2(a0.z, a0.w), z0 = pk2(c0.x, c0.y), w0 = pk2(c0.z, c0.w);
        const f32x2 x1 = pk2(a1.x, a1.y), y1 = pk2(a1.z, a1.w), z1 = pk2(c1.x, c1.y), w1 = pk2(c1.z, c1.w);
        f32x2 d0[Q], d1[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          d0[k] = ffma2(z0, MODE == 2 ? pz[k] : pk2(qz[k], qz[k]), w0);
          d1[k] = ffma2(z1, MODE == 2 ? pz[k] : pk2(qz[k], qz[k]), w1);
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          d0[k] = ffma2(y0, MODE == 2 ? py[k] : pk2(qy[k], qy[k]), d0[k]);
          d1[k] = ffma2(y1, MODE == 2 ? py[k] : pk2(qy[k], qy[k]), d1[k]);
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          d0[k] = ffma2(x0, MODE == 2 ? px[k] : pk2(qx[k], qx[k]), d0[k]);
          d1[k] = ffma2(x1, MODE == 2 ? px[k] : pk2(qx[k], qx[k]), d1[k]);
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          float l0, h0, l1, h1;
          up2(d0[k], l0, h0);
          up2(d1[k], l1, h1);
          if (MODE == 4) {  // 2-input min.f32, kept unfused
            float m0, m1, m2, m3;
            asm volatile("min.f32 %0, %1, %2;" : "=f"(m0) : "f"(l0), "f"(h0));
            asm volatile("min.f32 %0, %1, %2;" : "=f"(m1) : "f"(l1), "f"(h1));
            asm volatile("min.f32 %0, %1, %2;" : "=f"(m2) : "f"(m0), "f"(m1));
            asm volatile("min.f32 %0, %1, %2;" : "=f"(m3) : "f"(tm[k]), "f"(m2));
            tm[k] = m3;
          } else if (MODE == 5) {  // integer min of the bit patterns (timing only)
            const int a0 = min(__float_as_int(l0), __float_as_int(h0));
            const int a1 = min(__float_as_int(l1), __float_as_int(h1));
            tm[k] = __int_as_float(min(__float_as_int(tm[k]), min(a0, a1)));
          } else {
            tm[k] = fminf(fminf(tm[k], fminf(l0, h0)), fminf(l1, h1));
          }
        }
      }
      }
      const int sid = sub;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        if (MODE == 0) {
          b1[k] = fminf(b1[k], tm[k]);
        } else if (NET) {
          const bool lt1 = tm[k] < b1[k];
          const bool lt2 = tm[k] < b2[k];
          b3[k] = fminf(b3[k], fmaxf(b2[k], tm[k]));
          b2[k] = fminf(b2[k], fmaxf(b1[k], tm[k]));
          b1[k] = fminf(b1[k], tm[k]);
          const int s1 = s12[k] & 0xffff;
          s12[k] = (lt1 ? sid : s1) | ((lt1 ? s1 : (lt2 ? sid : (s12[k] >> 16))) << 16);
        } else {
          const bool lt1 = tm[k] < b1[k];
          const bool lt2 = tm[k] < b2[k];
          b3[k] = lt2 ? b2[k] : fminf(b3[k], tm[k]);
          const int s1 = s12[k] & 0xffff;
          const int s2 = lt1 ? s1 : (lt2 ? sid : (s12[k] >> 16));
          b2[k] = lt1 ? b1[k] : (lt2 ? tm[k] : b2[k]);
          b1[k] = lt1 ? tm[k] : b1[k];
          s12[k] = (lt1 ? sid : s1) | (s2 << 16);
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < Q; ++k) s += b1[k] + b2[k] + b3[k] + s12[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float4 *cand, *qin;
  float* out;
  cudaMalloc(&cand, kCand * sizeof(float4));
  {
    const int nq = sms * 8 * 128 * 16;
    float4* hq = new float4[nq];
    for (int i = 0; i < nq; ++i) hq[i] = make_float4(1e-4f * (i % 977), -2e-4f * (i % 511), 3e-4f * (i % 263), 0.f);
    cudaMalloc(&qin, nq * sizeof(float4));
    cudaMemcpy(qin, hq, nq * sizeof(float4), cudaMemcpyHostToDevice);
    delete[] hq;
  }
  cudaMalloc(&out, sizeof(float) * 128 * sms * 8);
  float4 h[kCand];
  for (int i = 0; i < kCand; ++i) h[i] = make_float4(0.001f * i, -0.002f * i, 0.0005f * i, 0.3f + 1e-4f * i);
  cudaMemcpy(cand, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 40;
  // Queries per thread (register blocking) for the hot loop alone.
  {
    auto run = [&](auto kern, int q, int per_sm) {
      const int blocks = sms * per_sm;
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        kern<<<blocks, 128>>>(cand, qin, out, reps);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      const double pairs = static_cast<double>(blocks) * 128 * q * kCand * reps;
      const double per_clk_sm = pairs / (best * 1e-3) / (static_cast<double>(sms) * clk * 1e3);
      printf("hot loop + top-3, Q=%d, %d CTAs/SM: %.2f pairs/clk/SM  FMA pipe %.2f\n", q, per_sm, per_clk_sm,
             per_clk_sm * 3 / 128);
    };
    run(loop_kernel<1, 8, 4, 8>, 8, 4);                 // select top-3, full subtile unroll
    run(loop_kernel<1, 8, 4, 8, 32, true>, 8, 4);       // min/max-network top-3 (the kernel's)
    run(loop_kernel<1, 8, 4, 16, 64, true>, 8, 4);      // top-3 per 64 candidates
    run(loop_kernel<0, 8, 4, 8>, 8, 4);                 // no top-3
    run(loop_kernel<1, 8, 3, 8, 32, true>, 8, 3);
    run(loop_kernel<1, 12, 3, 8, 32, true>, 12, 3);
    run(loop_kernel<1, 4, 6>, 4, 6);
    run(loop_kernel<1, 12, 2>, 12, 2);
    run(loop_kernel<1, 12, 3>, 12, 3);
    run(loop_kernel<1, 16, 2>, 16, 2);
  }
  const char* names[6] = {"hot loop only", "hot loop + top-3", "packed queries + top-3", "scalar FFMA + top-3",
                          "2-input min.f32 + top-3", "integer min + top-3"};
  for (int mode = 0; mode < 6; ++mode)
    for (int per_sm = 4; per_sm <= 4; ++per_sm) {
      const int blocks = sms * per_sm;
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) loop_kernel<0><<<blocks, 128>>>(cand, qin, out, reps);
        if (mode == 1) loop_kernel<1><<<blocks, 128>>>(cand, qin, out, reps);
        if (mode == 2) loop_kernel<2><<<blocks, 128>>>(cand, qin, out, reps);
        if (mode == 3) loop_kernel<3><<<blocks, 128>>>(cand, qin, out, reps);
        if (mode == 4) loop_kernel<4><<<blocks, 128>>>(cand, qin, out, reps);
        if (mode == 5) loop_kernel<5><<<blocks, 128>>>(cand, qin, out, reps);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      const double pairs = static_cast<double>(blocks) * 128 * 8 * kCand * reps;
      const double per_clk_sm = pairs / (best * 1e-3) / (static_cast<double>(sms) * clk * 1e3);
      printf("mode %d (%s) %d CTAs/SM: %.3f ms  %.2f pairs/clk/SM  FMA pipe %.2f  (8-FLOP: %.1f TFLOP/s at %d MHz)\n",
             mode, names[mode], per_sm, best, per_clk_sm, per_clk_sm * 3 / 128,
             8.0 * pairs / (best * 1e-3) / 1e12, clk / 1000);
    }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
