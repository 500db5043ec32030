// pr_kernels.cuh -- Parareal for linear IVPs (reference src/parareal.cpp:56-117;
// paper §4, Eq. (parareal1)):
//
//   y_{0,i+1}^{(k+1)} = G_i y_{0i}^{(k+1)} + (F_i - G_i) y_{0i}^{(k)}.
//
// Every propagator is a per-window stepper y <- T_i y + c_{i,n}, n = 1..S:
// a discrete one-step method has T_i = diag_i^{-1} sub_i and
// c_{i,n} = diag_i^{-1} rhs_{i,n}; the matrix-exponential propagator is one
// step with T_i = e^{delta_i L} and c = its forcing particular solution.
// Vectors are propagated (the paper's point: w_N is never formed).
//
//   pr_prep_kernel  : c_{i,n} = Minv_i rhs_{i,n}, once per problem
//   pr_fine_kernel  : one warp per window, all windows concurrently: the
//                     fine propagations F_i y^{(k)} and the old coarse terms
//                     G_i y^{(k)} (the expensive, parallel part)
//   pr_sweep_kernel : one warp, the sequential coarse sweep in i, plus the
//                     update norm max_i |y^{(k+1)} - y^{(k)}| and the scale
//                     max_i |y^{(k+1)}| for the stopping test
//
// Row r of the state lives in lane r % 32 (m <= 64: two rows per lane); T is
// staged transposed in shared memory so the lanes' reads are conflict-free.
#pragma once

namespace psg {

constexpr int kPrMaxM = 64;

struct PrStepper {
  int S;               // steps per window
  const double* T;     // p x m x m, row-major (window-major)
  const double* Minv;  // p x m x m
  const double* rhs;   // p x S x m method right-hand sides
  double* c;           // p x S x m: Minv rhs
  const int* mat;      // p: index of the window's T (windows with equal steps share one)
};

struct PrArgs {
  int m, p;
  PrStepper F, G;
  const double* y0;
  const double* old_inits;  // p x m
  double* new_inits;        // p x m
  double* fine;             // p x m: fine[i] = F_{i+1} old[i]
  double* gold;             // p x m: gold[i] = G_{i+1} old[i]
  double* norms;            // [0] update, [1] scale
  int with_fine;            // 0: pure coarse sweep (parareal_init)
};

__global__ void pr_prep_kernel(int m, int p, int S, const double* __restrict__ Minv, const int* __restrict__ mat,
                               const double* __restrict__ rhs, double* __restrict__ c) {
  const long task = (long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // (window, step)
  const int lane = threadIdx.x & 31;
  if (task >= (long)p * S) return;
  const long i = task / S;
  const double* M = Minv + (long)mat[i] * m * m;
  const double* g = rhs + task * m;
  for (int r = lane; r < m; r += 32) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __fma_rn(M[r * m + j], g[j], acc);
    c[task * m + r] = acc;
  }
}

// Stage T_i^T into shared memory (Tt[j * m + r] = T[r][j]).
__device__ __forceinline__ void pr_stage(double* Tt, const double* T, int m) {
  for (int e = threadIdx.x & 31; e < m * m; e += 32) {
    const int r = e / m, j = e - r * m;
    Tt[j * m + r] = T[e];
  }
  __syncwarp();
}

// S steps of y <- T y + c_n on the warp's state ys (shared, m doubles); c may
// be null (no forcing).  Four partial sums per row keep the FMA chains short.
__device__ __forceinline__ void pr_steps(double* ys, const double* Tt, const double* c, int m, int S) {
  const int lane = threadIdx.x & 31;
  const bool r0 = lane < m, r1 = lane + 32 < m;
  for (int n = 0; n < S; ++n) {
    double a0 = 0.0, a1 = 0.0;
    if (c) {
      const double* cn = c + (long)n * m;
      a0 = r0 ? cn[lane] : 0.0;
      a1 = r1 ? cn[lane + 32] : 0.0;
    }
    double s0[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
    int j = 0;
    for (; j + 4 <= m; j += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double yj = ys[j + u];
        if (r0) s0[u] = __fma_rn(Tt[(j + u) * m + lane], yj, s0[u]);
        if (r1) s1[u] = __fma_rn(Tt[(j + u) * m + lane + 32], yj, s1[u]);
      }
    }
    for (; j < m; ++j) {
      const double yj = ys[j];
      if (r0) s0[0] = __fma_rn(Tt[j * m + lane], yj, s0[0]);
      if (r1) s1[0] = __fma_rn(Tt[j * m + lane + 32], yj, s1[0]);
    }
    __syncwarp();
    if (r0) ys[lane] = __dadd_rn(__dadd_rn(s0[0], s0[1]) + __dadd_rn(s0[2], s0[3]), a0);
    if (r1) ys[lane + 32] = __dadd_rn(__dadd_rn(s1[0], s1[1]) + __dadd_rn(s1[2], s1[3]), a1);
    __syncwarp();
  }
}

struct PrSmem {
  double Tt[kPrMaxM * kPrMaxM];
  double y[kPrMaxM];
};

// Fine / old-coarse propagations, one CTA of NW warps per window i = 1..p-1:
// fine[i-1] = F_i old[i-1], gold[i-1] = G_i old[i-1].  Warp w owns columns
// [16w, 16w + 16) of T in registers (rows lane, lane + 32); partial row sums
// meet in shared memory, so one step is a 16-deep FMA chain plus a reduction.
struct PrFineSmem {
  double part[4][kPrMaxM];
  double y[kPrMaxM];
};

template <int NW>
__global__ void __launch_bounds__(32 * NW) pr_fine_kernel(PrArgs a) {
  __shared__ PrFineSmem S;
  const int i = blockIdx.x + 1, m = a.m;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (i >= a.p) return;
  const bool r0 = lane < m, r1 = lane + 32 < m;
  for (int h = 0; h < 2; ++h) {
    const PrStepper& P = h == 0 ? a.F : a.G;
    double* out = h == 0 ? a.fine : a.gold;
    const double* T = P.T + (long)P.mat[i - 1] * m * m;
    double t0[16], t1[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = 16 * w + jj;
      t0[jj] = (r0 && j < m) ? T[lane * m + j] : 0.0;
      t1[jj] = (r1 && j < m) ? T[(lane + 32) * m + j] : 0.0;
    }
    for (int r = threadIdx.x; r < m; r += 32 * NW) S.y[r] = a.old_inits[(long)(i - 1) * m + r];
    __syncthreads();
    const double* c = P.c ? P.c + (long)(i - 1) * P.S * m : nullptr;
    for (int n = 0; n < P.S; ++n) {
      double s0a = 0.0, s0b = 0.0, s1a = 0.0, s1b = 0.0;
#pragma unroll
      for (int jj = 0; jj < 16; jj += 2) {
        const double ya = S.y[16 * w + jj], yb = S.y[16 * w + jj + 1];
        s0a = __fma_rn(t0[jj], ya, s0a);
        s0b = __fma_rn(t0[jj + 1], yb, s0b);
        s1a = __fma_rn(t1[jj], ya, s1a);
        s1b = __fma_rn(t1[jj + 1], yb, s1b);
      }
      const double cn0 = (c && w == 0 && r0) ? c[(long)n * m + lane] : 0.0;
      const double cn1 = (c && w == 0 && r1) ? c[(long)n * m + lane + 32] : 0.0;
      if (NW == 1) {
        __syncwarp();
        if (r0) S.y[lane] = __dadd_rn(__dadd_rn(s0a, s0b), cn0);
        if (r1) S.y[lane + 32] = __dadd_rn(__dadd_rn(s1a, s1b), cn1);
        __syncwarp();
      } else {
        S.part[w][lane] = __dadd_rn(s0a, s0b);
        S.part[w][lane + 32] = __dadd_rn(s1a, s1b);
        __syncthreads();
        if (w == 0) {
          double v0 = S.part[0][lane], v1 = S.part[0][lane + 32];
#pragma unroll
          for (int q = 1; q < NW; ++q) {
            v0 = __dadd_rn(v0, S.part[q][lane]);
            v1 = __dadd_rn(v1, S.part[q][lane + 32]);
          }
          if (r0) S.y[lane] = __dadd_rn(v0, cn0);
          if (r1) S.y[lane + 32] = __dadd_rn(v1, cn1);
        }
        __syncthreads();
      }
    }
    for (int r = threadIdx.x; r < m; r += 32 * NW) out[(long)(i - 1) * m + r] = S.y[r];
    __syncthreads();
  }
}

// The sequential coarse sweep (one warp) and the stopping norms.
__global__ void __launch_bounds__(32) pr_sweep_kernel(PrArgs a) {
  extern __shared__ __align__(16) unsigned char pr_smem_raw[];
  PrSmem& S = *reinterpret_cast<PrSmem*>(pr_smem_raw);
  const int lane = threadIdx.x, m = a.m;
  double upd = 0.0, scale = 0.0;
  for (int r = lane; r < m; r += 32) {
    const double v = a.y0[r];
    a.new_inits[r] = v;
    S.y[r] = v;
    scale = fmax(scale, fabs(v));
  }
  __syncwarp();
  int staged = -1;
  // window i's fine / gold / old rows (lanes hold rows lane, lane + 32), loaded one window ahead
  auto load3 = [&](int i, double* v) {
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      const bool ok = i < a.p && r < m;
      v[3 * h + 0] = ok && a.with_fine ? a.fine[(long)(i - 1) * m + r] : 0.0;
      v[3 * h + 1] = ok && a.with_fine ? a.gold[(long)(i - 1) * m + r] : 0.0;
      v[3 * h + 2] = ok ? a.old_inits[(long)i * m + r] : 0.0;
    }
  };
  double cur[6], nxt[6];
  load3(1, cur);
  for (int i = 1; i < a.p; ++i) {
    load3(i + 1, nxt);
    const int mi = a.G.mat[i - 1];
    if (mi != staged) {
      pr_stage(S.Tt, a.G.T + (long)mi * m * m, m);
      staged = mi;
    }
    pr_steps(S.y, S.Tt, a.G.c ? a.G.c + (long)(i - 1) * a.G.S * m : nullptr, m, a.G.S);  // gnew = G_i y_new[i-1]
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      if (r >= m) continue;
      double v = S.y[r];
      if (a.with_fine)  // F + (gnew - gold) (src/parareal.cpp:81-86)
        v = __dadd_rn(cur[3 * h], __dsub_rn(v, cur[3 * h + 1]));
      a.new_inits[(long)i * m + r] = v;
      S.y[r] = v;
      upd = fmax(upd, fabs(__dsub_rn(v, cur[3 * h + 2])));
      scale = fmax(scale, fabs(v));
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 6; ++q) cur[q] = nxt[q];
  }
  for (int o = 16; o > 0; o >>= 1) {
    upd = fmax(upd, __shfl_xor_sync(0xffffffffu, upd, o));
    scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  }
  if (lane == 0) {
    a.norms[0] = upd;
    a.norms[1] = scale;
  }
}

// propagate(): one window, one stepper, one vector.
__global__ void __launch_bounds__(32) pr_apply_kernel(PrStepper P, int m, int i, const double* __restrict__ y,
                                                      double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char pr_smem_raw[];
  PrSmem& S = *reinterpret_cast<PrSmem*>(pr_smem_raw);
  const int lane = threadIdx.x;
  pr_stage(S.Tt, P.T + (long)P.mat[i - 1] * m * m, m);
  for (int r = lane; r < m; r += 32) S.y[r] = y[r];
  __syncwarp();
  pr_steps(S.y, S.Tt, P.c ? P.c + (long)(i - 1) * P.S * m : nullptr, m, P.S);
  for (int r = lane; r < m; r += 32) out[r] = S.y[r];
}

}  // namespace psg
