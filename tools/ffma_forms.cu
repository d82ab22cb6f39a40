// FP32 FMA issue-form microbenchmark (diagnostic): 3-register FFMA, packed
// FFMA2 (fma.rn.f32x2) and FFMA with a uniform-register operand, each as 16
// independent chains per thread on every SM.  Prints FMA/clk/SM and TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma_forms tools/ffma_forms.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_reg(float* out, int iters, const float* in) {
  float a = in[threadIdx.x & 31], b = in[32 + (threadIdx.x & 31)];
  float acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = __fmaf_rn(acc[k], a, b);
    a = __int_as_float(__float_as_int(a) ^ (i & 1));  // keep a, b per-thread registers
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_uniform(float* out, int iters, float a, float b) {
  float acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = __fmaf_rn(acc[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void ffma2_reg(float* out, int iters, const float* in) {
  const float a0 = in[threadIdx.x & 31], b0 = in[32 + (threadIdx.x & 31)];
  unsigned long long a = (static_cast<unsigned long long>(__float_as_uint(a0)) << 32) | __float_as_uint(a0 + 1.f);
  const unsigned long long b = (static_cast<unsigned long long>(__float_as_uint(b0)) << 32) | __float_as_uint(b0);
  unsigned long long acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = (static_cast<unsigned long long>(k) << 32) | threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = ffma2(acc[k], a, b);
    a ^= static_cast<unsigned long long>(i & 1);
  }
  unsigned long long s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(static_cast<unsigned>(s));
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int threads = 256, blocks = sms * 8, iters = 20000;
  float *out, *in;
  cudaMalloc(&out, sizeof(float) * threads * blocks);
  cudaMalloc(&in, 64 * sizeof(float));
  cudaMemset(in, 0, 64 * sizeof(float));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int form = 0; form < 3; ++form) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (form == 0) ffma_reg<<<blocks, threads>>>(out, iters, in);
      if (form == 1) ffma_uniform<<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f);
      if (form == 2) ffma2_reg<<<blocks, threads>>>(out, iters, in);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    const double fmas = 16.0 * iters * threads * static_cast<double>(blocks);
    const double per_clk_sm = fmas / (best * 1e-3) / (sms * clk * 1e3);
    printf("%-14s %8.3f ms  %7.2f FMA/clk/SM  %7.2f TFLOP/s (at %d MHz max)\n",
           form == 0 ? "FFMA 3-reg" : (form == 1 ? "FFMA uniform" : "FFMA2 3-reg"), best, per_clk_sm,
           2.0 * fmas / (best * 1e-3) / 1e12, clk / 1000);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
