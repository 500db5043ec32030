// tri_kernels.cuh -- sm_100a kernels of the partition method for scalar
// tridiagonal systems (reference Kind::Banded, s = r = 1; BASELINE configs 0
// and 1).
//
// Notation (one segment = one partition body, rows s .. s+L-1, with
// separator x_l = row s-1 on its left and x_r = row s+L on its right):
//   B y = f_body - a_s x_l e_0 - c_{s+L-1} x_r e_{L-1}
//   y = P + U x_l + V x_r,  P = B^-1 f,  U = B^-1(-a e_0),  V = B^-1(-c e_{L-1}).
// The reference's interface blocks (src/localfact.cpp:207-210) are, for the
// separator row t between segments i and i+1:
//   alpha2^(i) = b_t + a_t V^(i)_{L-1}        alpha1^(i+1) = c_t U^(i+1)_0
//   beta^(i)   = a_t U^(i)_{L-1}              gamma^(i+1)  = c_t V^(i+1)_0
// and the condensed right-hand sides (src/localfact.cpp:769-781) are
//   -v^T ghat = -a_t P^(i)_{L-1},  -w^T ghat = -c_t P^(i+1)_0.
//
// K1  tri_interface_kernel : the segment-end values (U0,V0,UL,VL | P0,PL).
//     Speculative mode sweeps only the first/last H rows (the fill-ins
//     z, w decay geometrically for the dominant generators);
//     exact mode sweeps the whole body.  One thread per segment end.
// K2  tri_assemble_*        : reduced tridiagonal system T (p-1 rows).
// K3  tri_segment_solve     : per-segment back-substitution
//     x_body = B^-1(f - a x_l e_0 - c x_r e_{L-1}) by a 64-thread
//     two-level partition ("Laszlo") elimination with TMA-staged rows,
//     conflict-free odd-stride shared-memory walks and an in-CTA PCR on the
//     64 chunk interfaces; also the certificate (separator-row residuals) and
//     the direct solve of small reduced systems (nseg = 1).
#pragma once

#include "psg_common.cuh"

namespace psg {

struct TriRows {
  RowArr a, b, c;  // sub (coefficient of row r-1), diagonal, super (coefficient of row r+1)
};

// ----------------------------------------------------------------------------
// K1: segment-end interface values
// ----------------------------------------------------------------------------
// out_mat[4*seg + {0,1,2,3}] = U0, V0, UL, VL   (when WITH_MAT)
// out_rhs[2*seg + {0,1}]     = P0, PL           (when WITH_RHS)
template <bool WITH_MAT, bool WITH_RHS>
__global__ void __launch_bounds__(128) tri_interface_kernel(TriRows A, RowArr F, const int* __restrict__ seg_start,
                                                             const int* __restrict__ seg_len, int nseg, int H,
                                                             double* __restrict__ out_mat,
                                                             double* __restrict__ out_rhs) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int seg = idx >> 1;
  if (seg >= nseg) return;
  const int end = idx & 1;
  const long s = seg_start[seg];
  const int L = seg_len[seg];
  const int h = (H <= 0 || 2 * H >= L) ? L : H;
  if (end == 0) {
    // Bottom-up (UL) sweep over rows h-1 .. 0: row 0 becomes
    //   e y_0 + a_s x_l = g + hv x_r.
    long r = s + h - 1;
    double e = row_at(A.b, r);
    double g = WITH_RHS ? row_at(F, r) : 0.0;
    double hv = (h == L) ? -row_at(A.c, r) : 0.0;
#pragma unroll 4
    for (int j = h - 2; j >= 0; --j) {
      r = s + j;
      const double cj = row_at(A.c, r);
      const double an = row_at(A.a, r + 1);
      const double mu = cj / e;
      e = fma(-mu, an, row_at(A.b, r));
      if (WITH_RHS) g = fma(-mu, g, row_at(F, r));
      if (WITH_MAT) hv = -mu * hv;
    }
    const double inv = 1.0 / e;
    if (WITH_MAT) {
      out_mat[4 * seg + 0] = -row_at(A.a, s) * inv;
      out_mat[4 * seg + 1] = hv * inv;
    }
    if (WITH_RHS) out_rhs[2 * seg + 0] = g * inv;
  } else {
    // Top-down (LU) sweep over rows L-h .. L-1: row L-1 becomes
    //   d y_{L-1} + c x_r = g + hu x_l.
    const int j0 = L - h;
    long r = s + j0;
    double d = row_at(A.b, r);
    double g = WITH_RHS ? row_at(F, r) : 0.0;
    double hu = (j0 == 0) ? -row_at(A.a, r) : 0.0;
#pragma unroll 4
    for (int j = j0 + 1; j < L; ++j) {
      r = s + j;
      const double aj = row_at(A.a, r);
      const double cp = row_at(A.c, r - 1);
      const double l = aj / d;
      d = fma(-l, cp, row_at(A.b, r));
      if (WITH_RHS) g = fma(-l, g, row_at(F, r));
      if (WITH_MAT) hu = -l * hu;
    }
    const double inv = 1.0 / d;
    if (WITH_MAT) {
      out_mat[4 * seg + 2] = hu * inv;
      out_mat[4 * seg + 3] = -row_at(A.c, s + L - 1) * inv;
    }
    if (WITH_RHS) out_rhs[2 * seg + 1] = g * inv;
  }
}

// ----------------------------------------------------------------------------
// K2: reduced system assembly.  Separator j sits at row t = start_j + len_j.
//   Tsub[j]  = a_t UL_j          (coefficient of x_{j-1})
//   Tdiag[j] = b_t + a_t VL_j + c_t U0_{j+1}
//   Tsup[j]  = c_t V0_{j+1}      (coefficient of x_{j+1})
//   rhs[j]   = f_t - a_t PL_j - c_t P0_{j+1}
// ----------------------------------------------------------------------------
__global__ void tri_assemble_matrix_kernel(TriRows A, const int* __restrict__ seg_start,
                                           const int* __restrict__ seg_len, int nsep,
                                           const double* __restrict__ mat, double* __restrict__ Tsub,
                                           double* __restrict__ Tdiag, double* __restrict__ Tsup) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nsep) return;
  const long t = (long)seg_start[j] + seg_len[j];
  const double a = row_at(A.a, t), b = row_at(A.b, t), c = row_at(A.c, t);
  Tsub[j] = a * mat[4 * j + 2];
  Tdiag[j] = fma(c, mat[4 * (j + 1) + 0], fma(a, mat[4 * j + 3], b));
  Tsup[j] = c * mat[4 * (j + 1) + 1];
}

__global__ void tri_assemble_rhs_kernel(TriRows A, RowArr F, const int* __restrict__ seg_start,
                                        const int* __restrict__ seg_len, int nsep,
                                        const double* __restrict__ rhs_in, double* __restrict__ rhs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nsep) return;
  const long t = (long)seg_start[j] + seg_len[j];
  const double a = row_at(A.a, t), c = row_at(A.c, t);
  rhs[j] = fma(-c, rhs_in[2 * (j + 1) + 0], fma(-a, rhs_in[2 * j + 1], row_at(F, t)));
}

// ----------------------------------------------------------------------------
// K3: per-segment solve.  CTA = NT threads = one segment of <= M*NT rows;
// thread t owns body rows [tM, tM+M) (M odd => the stride-M shared-memory
// walk of a warp touches 16 distinct 8-byte bank pairs: 2 wavefronts, the
// minimum for 64-bit loads).
// ----------------------------------------------------------------------------
struct TriSolveArgs {
  TriRows A;
  RowArr F;
  const int* seg_start;
  const int* seg_len;
  int nseg;
  const double* xsep;  // nseg-1 separator values (NULL when nseg == 1)
  double* x;           // output, row r at x[r]
  // certificate (level 1 only; NULL disables)
  double2* partR;
  double2* partL;
  int* counters;
  DevStatus* status;
};

template <int M, int NT>
struct TriSmem {
  static constexpr int LCAP = M * NT + 2;   // body rows + both separators
  static constexpr int ROW = LCAP + 2;      // + alignment shift, even
  static constexpr int BYTES = (4 * ROW + 8 * NT + 2 * NT) * 8 + 16;
};

__device__ __forceinline__ void cert_combine(const double2* partR, const double2* partL, int j, DevStatus* st) {
  const double2 R = __ldcg(partR + j);
  const double2 Lp = __ldcg(partL + j);
  const double v = R.x + Lp.x;
  const double a = R.y + Lp.y;
  double w = a > 0.0 ? fabs(v) / a : (v != 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0);
  status_cert(st, w);
}

template <int M, int NT>
__global__ void __launch_bounds__(NT) tri_segment_solve_kernel(TriSolveArgs args) {
  static_assert(M % 2 == 1 && M >= 3, "M must be odd and >= 3");
  using SM = TriSmem<M, NT>;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int seg = blockIdx.x;
  const long s = args.seg_start[seg];
  const int L = args.seg_len[seg];

  double* sA;
  double* sB;
  double* sC;
  double* sF;
  double* pcr = smem + 4 * SM::ROW;  // 2 x 4 x NT
  double* sx = pcr + 8 * NT;         // 2 x NT scratch (E rows, F values)
  __shared__ double* bufs[4];
  if (tid == 0) {
    mbar_init(&bar, 1);
    uint32_t tx = 0;
    const long r0 = s - 1, r1 = s + L + 1;
    bufs[0] = stage_rows(args.A.a, r0, r1, smem + 0 * SM::ROW, &bar, &tx);
    bufs[1] = stage_rows(args.A.b, r0, r1, smem + 1 * SM::ROW, &bar, &tx);
    bufs[2] = stage_rows(args.A.c, r0, r1, smem + 2 * SM::ROW, &bar, &tx);
    bufs[3] = stage_rows(args.F, r0, r1, smem + 3 * SM::ROW, &bar, &tx);
    mbar_arrive_expect_tx(&bar, tx);
  }
  const double xl = (seg > 0) ? args.xsep[seg - 1] : 0.0;
  const double xr = (seg < args.nseg - 1) ? args.xsep[seg] : 0.0;
  __syncthreads();
  mbar_wait(&bar, 0);
  sA = bufs[0];
  sB = bufs[1];
  sC = bufs[2];
  sF = bufs[3];

  // ---- chunk elimination: every row j of the chunk ends as
  //      ap[j] * y_first + y_j + cp[j] * y_last = dp[j]
  //      (row 0: ap*y_{prev chunk last} + y_0 + cp*y_last; row M-1: ap*y_0 + y_{M-1} + cp*y_{next first})
  double ap[M], cp[M], dp[M];
  const int q0 = tid * M;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const int q = q0 + j;
    const bool valid = q < L;
    double a = valid ? sA[1 + q] : 0.0;
    const double b = valid ? sB[1 + q] : 1.0;
    double c = valid ? sC[1 + q] : 0.0;
    double f = valid ? sF[1 + q] : 0.0;
    if (q == 0) {
      f = fma(-a, xl, f);
      a = 0.0;
    }
    if (q == L - 1) {
      f = fma(-c, xr, f);
      c = 0.0;
    }
    if (j < 2) {
      const double r = 1.0 / b;
      ap[j] = a * r;
      cp[j] = c * r;
      dp[j] = f * r;
    } else {
      const double r = 1.0 / fma(-a, cp[j - 1], b);
      dp[j] = r * fma(-a, dp[j - 1], f);
      ap[j] = -r * a * ap[j - 1];
      cp[j] = r * c;
    }
  }
#pragma unroll
  for (int j = M - 3; j >= 1; --j) {
    dp[j] = fma(-cp[j], dp[j + 1], dp[j]);
    ap[j] = fma(-cp[j], ap[j + 1], ap[j]);
    cp[j] = -cp[j] * cp[j + 1];
  }
  {
    const double r = 1.0 / fma(-cp[0], ap[1], 1.0);
    dp[0] = r * fma(-cp[0], dp[1], dp[0]);
    ap[0] = r * ap[0];
    cp[0] = -r * cp[0] * cp[1];
  }

  // ---- chunk interfaces: eliminate the E (last-row) unknowns, giving one
  //      tridiagonal row per thread in the F (first-row) unknowns.
  double* sEa = sx;  // reuse: E rows need 3 arrays -> use pcr buffer 1 region
  double* eA = pcr + 4 * NT;
  double* eC = eA + NT;
  double* eD = eC + NT;
  eA[tid] = ap[M - 1];
  eC[tid] = cp[M - 1];
  eD[tid] = dp[M - 1];
  __syncthreads();
  double al, be, ga, de;
  {
    const double pa = tid > 0 ? eA[tid - 1] : 0.0;
    const double pc = tid > 0 ? eC[tid - 1] : 0.0;
    const double pd = tid > 0 ? eD[tid - 1] : 0.0;
    al = -ap[0] * pa;
    be = 1.0 - ap[0] * pc - cp[0] * ap[M - 1];
    ga = -cp[0] * cp[M - 1];
    de = dp[0] - ap[0] * pd - cp[0] * dp[M - 1];
  }
  (void)sEa;
  // ---- parallel cyclic reduction over the NT F-rows (double-buffered).
  int buf = 0;
#pragma unroll
  for (int st = 1; st < NT; st <<= 1) {
    double* P = pcr + buf * 4 * NT;
    P[tid] = al;
    P[NT + tid] = be;
    P[2 * NT + tid] = ga;
    P[3 * NT + tid] = de;
    __syncthreads();
    double la = 0.0, lb = 1.0, lg = 0.0, ld = 0.0, ha = 0.0, hb = 1.0, hg = 0.0, hd = 0.0;
    if (tid - st >= 0) {
      la = P[tid - st];
      lb = P[NT + tid - st];
      lg = P[2 * NT + tid - st];
      ld = P[3 * NT + tid - st];
    }
    if (tid + st < NT) {
      ha = P[tid + st];
      hb = P[NT + tid + st];
      hg = P[2 * NT + tid + st];
      hd = P[3 * NT + tid + st];
    }
    const double k1 = al / lb;
    const double k2 = ga / hb;
    al = -k1 * la;
    ga = -k2 * hg;
    be = be - k1 * lg - k2 * ha;
    de = de - k1 * ld - k2 * hd;
    buf ^= 1;
  }
  const double Fv = de / be;
  sx[tid] = Fv;
  __syncthreads();
  const double Fn = tid + 1 < NT ? sx[tid + 1] : 0.0;
  const double Ev = dp[M - 1] - ap[M - 1] * Fv - cp[M - 1] * Fn;

  // ---- chunk back-substitution, finite check, stage y over f.
  bool finite = true;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const int q = q0 + j;
    double y;
    if (j == 0)
      y = Fv;
    else if (j == M - 1)
      y = Ev;
    else
      y = dp[j] - ap[j] * Fv - cp[j] * Ev;
    if (q < L) {
      finite &= isfinite(y);
      sF[1 + q] = y;
    }
  }
  if (!finite && args.status) status_nonfinite(args.status, seg);
  __syncthreads();

  // ---- coalesced write-back of the body (and the right separator).
  double* xo = args.x + s;
  for (int q = tid; q < L; q += NT) xo[q] = sF[1 + q];

  if (tid == 0 && seg < args.nseg - 1) args.x[s + L] = xr;

  // ---- certificate: componentwise backward error of the separator rows,
  //      combined by whichever neighbouring CTA arrives second.
  if (tid == 0 && args.counters) {
    const double y0 = sF[1], yL = sF[L];
    if (seg < args.nseg - 1) {
      const double aR = sA[L + 1], bR = sB[L + 1], fR = sF[L + 1];
      const double t1 = aR * yL, t2 = bR * xr;
      args.partR[seg] = make_double2(fR - t1 - t2, fabs(fR) + fabs(t1) + fabs(t2));
      __threadfence();
      if (atomicAdd(args.counters + seg, 1) == 1) {
        __threadfence();
        cert_combine(args.partR, args.partL, seg, args.status);
        args.counters[seg] = 0;
      }
    }
    if (seg > 0) {
      const double t3 = sC[0] * y0;
      args.partL[seg - 1] = make_double2(-t3, fabs(t3));
      __threadfence();
      if (atomicAdd(args.counters + seg - 1, 1) == 1) {
        __threadfence();
        cert_combine(args.partR, args.partL, seg - 1, args.status);
        args.counters[seg - 1] = 0;
      }
    }
  }
}

}  // namespace psg
