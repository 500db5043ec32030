// Host cost of the production loop's C-ABI calls (psg_refactor +
// psg_solve_async) on the config-0 system: per-call wall time, no Python.
//   g++ -O2 -Iinclude tools/host_calls.cpp -Lpaper_0912_3678_b200 -lpsg -lcudart ...
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include "psg.h"

int main() {
  const int n = 1 << 20, p = 1024;
  char err[512];
  double *data, *f, *x;
  cudaMalloc(&data, sizeof(double) * (3 * (size_t)n - 2));
  cudaMalloc(&f, sizeof(double) * n);
  cudaMalloc(&x, sizeof(double) * n);
  if (psg_generate_config(0, n, 1, data, nullptr, f, nullptr, err, sizeof err)) return printf("gen: %s\n", err), 1;
  psg_desc A{PSG_BANDED, n, 1, 1, 1, data, 3 * (size_t)n - 2, nullptr, 0, 0, 1};
  psg_handle* h = nullptr;
  if (psg_factor(&A, p, PSG_LU, 1e-8, nullptr, &h, err, sizeof err)) return printf("factor: %s\n", err), 1;
  for (int i = 0; i < 50; ++i) {
    psg_refactor(h, &A, nullptr, err, sizeof err);
    psg_solve_async(h, f, x, 0, nullptr, err, sizeof err);
  }
  psg_sync(h, nullptr, err, sizeof err);
  cudaDeviceSynchronize();
  using clk = std::chrono::steady_clock;
  const int N = 500;
  double tr = 0, ts = 0;
  auto t0 = clk::now();
  for (int i = 0; i < N; ++i) {
    auto a = clk::now();
    psg_refactor(h, &A, nullptr, err, sizeof err);
    auto b = clk::now();
    psg_solve_async(h, f, x, 0, nullptr, err, sizeof err);
    auto c = clk::now();
    tr += std::chrono::duration<double, std::micro>(b - a).count();
    ts += std::chrono::duration<double, std::micro>(c - b).count();
  }
  auto t1 = clk::now();
  psg_sync(h, nullptr, err, sizeof err);
  cudaDeviceSynchronize();
  auto t2 = clk::now();
  printf("psg_refactor %.1f us, psg_solve_async %.1f us per call; loop %.1f us/step enqueue, %.1f us/step total\n",
         tr / N, ts / N, std::chrono::duration<double, std::micro>(t1 - t0).count() / N,
         std::chrono::duration<double, std::micro>(t2 - t0).count() / N);
  // bare launch cost for comparison
  cudaEvent_t e;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  auto u0 = clk::now();
  for (int i = 0; i < N; ++i) cudaEventRecord(e, 0);
  auto u1 = clk::now();
  printf("cudaEventRecord %.2f us\n", std::chrono::duration<double, std::micro>(u1 - u0).count() / N);
  psg_release(h);
  return 0;
}
