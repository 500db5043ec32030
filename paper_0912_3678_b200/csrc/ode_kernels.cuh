// ode_kernels.cuh -- the time-parallel IVP trajectory as one BVP-layout BABD
// (reference src/odeparallel.cpp:183-233, solve_ivp_parallel; paper §3,
// Eq. (My)).  The one-step recursion  diag_w y_k = sub_w y_{k-1} + g_k  of
// all p N steps, closed by y_0 = y0, is expanded in HBM from the p window
// blocks (diag_w, sub_w) and the (p N + 1) m right-hand-side samples, so the
// host uploads O(p m^2 + p N m) doubles instead of the (p N) 2 MB^2 matrix.
// Dimensions m <= 8 are padded to MB in {2, 4, 8} with inert components
// (padding rows [-I | I], zero right-hand side); trajectories shorter than
// 64 steps get identity steps y_{k+1} = y_k appended.  Both kernels are
// pure streaming writes (HBM-bound): grid-stride, coalesced on the output.
#pragma once

#include <cstdint>

// Block row 0 = I (MB x MB); block row k + 1 (k < nsteps) = [-sub_w | diag_w]
// with w = k / N for k < p N (identity step otherwise); f = [y0 | g_1 .. g_pN]
// padded per block.  win = p x (diag, sub), each m x m row-major.
template <int MB>
__global__ void __launch_bounds__(256) ode_assemble_kernel(int m, long long steps, long long nsteps, int N,
                                                            const double* __restrict__ win,
                                                            const double* __restrict__ g, double* __restrict__ data,
                                                            double* __restrict__ f) {
  constexpr int BW = 2 * MB * MB;     // doubles per block row (a power of two)
  constexpr int RPB = 256 / BW > 0 ? 256 / BW : 1;  // block rows per 256 threads
  const int e = threadIdx.x % BW, rl = threadIdx.x / BW;
  const int i = e / (2 * MB), jj = e % (2 * MB);
  const bool left = jj < MB;
  const int j = left ? jj : jj - MB;
  const bool real = i < m && j < m;
  const double pad = (i == j) ? (left ? -1.0 : 1.0) : 0.0;
  if (blockIdx.x == 0 && threadIdx.x < MB * MB) data[threadIdx.x] = (threadIdx.x / MB == threadIdx.x % MB) ? 1.0 : 0.0;
  // block row k + 1 of the BABD (k = step index): one 32-bit window lookup per element
  for (long long k = (long long)blockIdx.x * RPB + rl; k < nsteps; k += (long long)gridDim.x * RPB) {
    double v = pad;
    if (k < steps && real) {
      const int w = (int)((unsigned)k / (unsigned)N);
      const double* W = win + (long long)w * 2 * m * m;
      v = left ? -W[m * m + i * m + j] : W[i * m + j];
    }
    data[MB * MB + k * BW + e] = v;
  }
  const long long nf = (nsteps + 1) * MB;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nf; t += stride) {
    const long long b = t / MB;
    const int q = (int)(t % MB);
    f[t] = (b <= steps && q < m) ? g[b * m + q] : 0.0;
  }
}

// Trajectory (steps + 1) x m from the padded solution (steps + 1) x MB.
template <int MB>
__global__ void ode_unpad_kernel(int m, long long steps, const double* __restrict__ x, double* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long total = (steps + 1) * m;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const long long b = t / m;
    out[t] = x[b * MB + (t - b * m)];
  }
}
