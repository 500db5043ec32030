// Dependent-issue latencies on the device (cycles per dependent instruction, one warp,
// clock64 around a long dependent chain): DFMA, DADD, 64-bit shuffle, LDS.64, MUFU.RCP64H + 2 Newton steps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat_probe tools/lat_probe.cu && /tmp/lat_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x] = threadIdx.x ^ 1;
  sm[threadIdx.x + 32] = 0.0;
  __syncwarp();
  double x = a + threadIdx.x;
  int idx = threadIdx.x;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = fma(x, a, b);
    if (OP == 1) x = x + b;
    if (OP == 2) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    if (OP == 3) {
      idx = (int)sm[idx & 31];
      x += idx;
    }
    if (OP == 4) x = fast_rcp(x);
    if (OP == 5) x = fma(x, a, __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 7, 8));
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x + idx;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMallocManaged(&cyc, 8);
  const int n = 4096;
  const char* names[] = {"DFMA dependent", "DADD dependent", "SHFL.64 dependent", "LDS.64 -> int -> LDS", "rcp.approx + 2 Newton",
                         "width-8 SHFL.64 + DFMA"};
  for (int rep = 0; rep < 2; ++rep) {
    chain<0><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); cudaDeviceSynchronize(); if (rep) printf("%-28s %6.1f cycles\n", names[0], double(*cyc) / n);
    chain<1><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); cudaDeviceSynchronize(); if (rep) printf("%-28s %6.1f cycles\n", names[1], double(*cyc) / n);
    chain<2><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); cudaDeviceSynchronize(); if (rep) printf("%-28s %6.1f cycles\n", names[2], double(*cyc) / n);
    chain<3><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); cudaDeviceSynchronize(); if (rep) printf("%-28s %6.1f cycles\n", names[3], double(*cyc) / n);
    chain<4><<<1, 32>>>(out, cyc, 1.5, 1e-9, n); cudaDeviceSynchronize(); if (rep) printf("%-28s %6.1f cycles\n", names[4], double(*cyc) / n);
    chain<5><<<1, 32>>>(out, cyc, 0.5, 1e-9, n); cudaDeviceSynchronize(); if (rep) printf("%-28s %6.1f cycles\n", names[5], double(*cyc) / n);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
