// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
// Dependent-chain latency of a few instruction classes on this GPU (cycles),
// one thread: DADD, DMUL, DFMA, FFMA, LDS.64 + DADD, DP sqrt, DP division.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = a + threadIdx.x;
  __syncthreads();
  if (threadIdx.x) return;
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, b);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, b, a);
  long long t3 = clock64();
  float f = (float)x;
  for (int i = 0; i < n; ++i) f = __fmaf_rn(f, (float)b, (float)a);
  long long t4 = clock64();
  int idx = 0;
  for (int i = 0; i < n; ++i) {
    const double v = sm[idx & 63];
    x = __dadd_rn(x, v);
    idx = (int)(v) + i;
  }
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x = b / (x + 1.0);
  long long t7 = clock64();
  out[0] = x + f;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6;
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  const int n = 4096;
  lat<<<1, 64>>>(o, c, 1.0000001, 0.9999999, n);
  lat<<<1, 64>>>(o, c, 1.0000001, 0.9999999, n);
  long long h[7];
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  const char* nm[7] = {"DADD", "DMUL", "DFMA", "FFMA", "LDS.64+DADD+F2I", "DP sqrt(+add)", "DP div(+add)"};
  for (int i = 0; i < 7; ++i) printf("%-18s %.1f cycles\n", nm[i], (double)h[i] / n);
  return 0;
}
