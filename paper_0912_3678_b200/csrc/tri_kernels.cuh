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

#include <climits>

#include "psg_common.cuh"

namespace psg {

__device__ __forceinline__ double b_minus(double b, double x, double y) { return (b - x) - y; }

struct TriRows {
  RowArr a, b, c;  // sub (coefficient of row r-1), diagonal, super (coefficient of row r+1)
};

// Segment i = rows [start, start+len) with one separator row after it.
// Uniform maps use the reference plan formula (src/partition.cpp:94-104 with
// k = 1): len = base + (i < rem), start = i*(base+1) + min(i, rem); refined
// plans pass explicit arrays.
struct SegMap {
  int nseg, base, rem;
  const int* start;
  const int* len;
};

__device__ __forceinline__ void seg_of(const SegMap& S, int i, long& s, int& L) {
  if (S.start) {
    s = S.start[i];
    L = S.len[i];
  } else {
    L = S.base + (i < S.rem ? 1 : 0);
    s = (long)i * (S.base + 1) + (i < S.rem ? i : S.rem);
  }
}

// ----------------------------------------------------------------------------
// K1: segment-end interface values
// ----------------------------------------------------------------------------
// out_mat[4*seg + {0,1,2,3}] = U0, V0, UL, VL   (when WITH_MAT)
// out_rhs[2*seg + {0,1}]     = P0, PL           (when WITH_RHS)
template <bool WITH_MAT, bool WITH_RHS>
__global__ void __launch_bounds__(128) tri_interface_kernel(TriRows A, RowArr F, SegMap S, int H,
                                                             double* __restrict__ out_mat,
                                                             double* __restrict__ out_rhs) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int seg = idx >> 1;
  if (seg >= S.nseg) return;
  const int end = idx & 1;
  long s;
  int L;
  seg_of(S, seg, s, L);
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
__global__ void tri_assemble_matrix_kernel(TriRows A, SegMap S,
                                           const double* __restrict__ mat, double* __restrict__ Tsub,
                                           double* __restrict__ Tdiag, double* __restrict__ Tsup) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= S.nseg - 1) return;
  long s0;
  int L0;
  seg_of(S, j, s0, L0);
  const long t = s0 + L0;
  const double a = row_at(A.a, t), b = row_at(A.b, t), c = row_at(A.c, t);
  Tsub[j] = a * mat[4 * j + 2];
  Tdiag[j] = fma(c, mat[4 * (j + 1) + 0], fma(a, mat[4 * j + 3], b));
  Tsup[j] = c * mat[4 * (j + 1) + 1];
}

__global__ void tri_assemble_rhs_kernel(TriRows A, RowArr F, SegMap S,
                                        const double* __restrict__ rhs_in, double* __restrict__ rhs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= S.nseg - 1) return;
  long s0;
  int L0;
  seg_of(S, j, s0, L0);
  const long t = s0 + L0;
  const double a = row_at(A.a, t), c = row_at(A.c, t);
  rhs[j] = fma(-c, rhs_in[2 * (j + 1) + 0], fma(-a, rhs_in[2 * j + 1], row_at(F, t)));
}


// ----------------------------------------------------------------------------
// Speculative interface, one warp per separator row t between
// segments j and j+1.  Truncate both adjacent bodies to their H = 32 rows next
// to t: the first row of the inverse of the leading block of segment j+1 and
// the last row of the inverse of the trailing block of segment j follow from
// two 32-row transposed solves (warp PCR, one row per lane).  Because the
// far-corner entries of a body inverse are O(rho^L) (exactly 0.0 in fp64 for
// the BASELINE generators, where the reference's beta/gamma also vanish), the
// speculative reduced matrix is diagonal:
//   Tdiag_t = b_t - a_t c_{t-1} v_31 - c_t a_{t+1} w_0
//   x_t     = ( f_t - a_t sum_i v_i f_{t-32+i} - c_t sum_i w_i f_{t+1+i} ) / Tdiag_t
// The factor stores the 65 weights of that dot product; the solve is one
// coalesced dot product per separator.  The certificate (separator residuals
// after the exact body solves) decides whether the speculation stands.
// ----------------------------------------------------------------------------
constexpr int kHalo = 32;

// Solve the 32x32 tridiagonal system held one row per lane
//   lo*y_{i-1} + di*y_i + up*y_{i+1} = r   (out-of-block couplings zeroed)
// by 5 normalised parallel-cyclic-reduction steps.  Returns y_lane.
__device__ __forceinline__ double warp_tri_pcr(double lo, double di, double up, double r) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double inv = fast_rcp(di);
  lo *= inv;
  up *= inv;
  r *= inv;
#pragma unroll
  for (int st = 1; st < 32; st <<= 1) {
    double la = __shfl_up_sync(FULL, lo, st), lu = __shfl_up_sync(FULL, up, st), lr = __shfl_up_sync(FULL, r, st);
    double ha = __shfl_down_sync(FULL, lo, st), hu = __shfl_down_sync(FULL, up, st),
           hr = __shfl_down_sync(FULL, r, st);
    if (lane < st) la = lu = lr = 0.0;
    if (lane + st >= 32) ha = hu = hr = 0.0;
    inv = fast_rcp(1.0 - lo * lu - up * ha);
    const double nr = r - lo * lr - up * hr;
    lo = -lo * la * inv;
    up = -up * hu * inv;
    r = nr * inv;
  }
  return r;
}

// Speculative separators in one pass over the 65-row window of every
// separator t (rows t-32 .. t+32 of a, b, c and, when the right-hand side is
// known, f).  Trailing block (rows t-32 .. t-1): the top-down Thomas sweep
//   d_k = b_k - l_k c_{k-1},  l_k = a_k / d_{k-1},  g_k = f_k - l_k g_{k-1}
// gives v_31 = 1/d_31 and v . f = g_31 / d_31 (v = last row of the block's
// inverse: the forward sweep IS the dot product, no weights are formed).
// Leading block (rows t+1 .. t+32): the same sweep bottom-up,
//   e_k = b_k - mu_k a_{k+1},  mu_k = c_k / e_{k+1},  h_k = f_k - mu_k h_{k+1}
// gives w_0 = 1/e_0 and w . f = h_0 / e_0.  Then
//   Tdiag_t = b_t - a_t c_{t-1} / d_31 - c_t a_{t+1} / e_0
//   x_t     = (f_t - a_t g_31 / d_31 - c_t h_0 / e_0) / Tdiag_t.
// One warp = 16 separators: lanes < 16 sweep the trailing blocks, lanes >= 16
// the leading ones (the same recurrence read in opposite row orders); every
// (array, separator) window is one TMA bulk copy, all in flight on one
// mbarrier.  WITH_F = false: Tdiag only (the factor alone).  Separators
// [jbase, jend) (the host path solves in row chunks).  The factor is lazy:
// a refactor followed by a solve is this single launch.
constexpr int kFacSeps = 16;             // separators per warp (one per half-warp lane pair)
constexpr int kWin = 2 * kHalo + 1;      // window rows t-32 .. t+32
constexpr int kFacPitch = 70;            // per-(array, separator) window slot: 65 rows + staging slack,
                                         // 16-byte multiple; 70 = 6 mod 16 keeps lane conflicts 2-way

template <bool WITH_F>
__global__ void __launch_bounds__(32) tri_spec_fused_kernel(TriRows A, RowArr F, SegMap S, double* __restrict__ xsep,
                                                            double* __restrict__ Tdiag, DevStatus* reset, int jbase,
                                                            int jend) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NA = WITH_F ? 4 : 3;
  __shared__ __align__(16) double tile[NA * kFacSeps * kFacPitch];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int shifts[NA * kFacSeps];
  if (WITH_F) pdl_trigger();  // K3 may launch and stage its rows while the separators finish
  const int lane = threadIdx.x;
  if (reset && blockIdx.x == 0 && lane < kCertSlots) reset->cert_bits[lane] = 0ull;  // first kernel of the solve
  if (reset && blockIdx.x == 0 && lane == 0) {
    reset->bad_seg = 0x7fffffff;
    reset->pivot_seg = 0x7fffffff;
  }
  const int j0 = jbase + blockIdx.x * kFacSeps;
  if (j0 >= jend) {
    pdl_wait();
    return;
  }
  const int nj = min(kFacSeps, jend - j0);
  const int jj = lane & (kFacSeps - 1);
  long tme;
  {
    long s0;
    int L0;
    seg_of(S, min(j0 + jj, jend - 1), s0, L0);
    tme = s0 + L0;
  }
  // ---- windows -> shared: task = (array x, separator q), one bulk copy each
  if (lane == 0) mbar_init(&bar, NA * kFacSeps);
  __syncwarp();
  for (int task = lane; task < NA * kFacSeps; task += 32) {
    const int x = task / kFacSeps;  // separator task % kFacSeps == lane & 15
    const RowArr X = x == 0 ? A.a : x == 1 ? A.b : x == 2 ? A.c : F;
    uint32_t tx = 0;
    shifts[task] = stage_issue(X, tme - kHalo, tme + kHalo + 1, tile + task * kFacPitch, &bar, &tx);
    mbar_arrive_expect_tx(&bar, tx);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  const double* wA = tile + (0 * kFacSeps + jj) * kFacPitch + 1 + shifts[0 * kFacSeps + jj];
  const double* wB = tile + (1 * kFacSeps + jj) * kFacPitch + 1 + shifts[1 * kFacSeps + jj];
  const double* wC = tile + (2 * kFacSeps + jj) * kFacPitch + 1 + shifts[2 * kFacSeps + jj];
  const double* wF = WITH_F ? tile + (3 * kFacSeps + jj) * kFacPitch + 1 + shifts[3 * kFacSeps + jj] : nullptr;
  // ---- one sweep per lane: lanes < 16 the trailing block (window rows 0..31
  //      downwards), lanes >= 16 the leading block (rows 64..33 upwards)
  const bool trail = lane < kFacSeps;
  const double* Nm = trail ? wA : wC;  // multiplier numerator (a | c)
  const double* Qc = trail ? wC : wA;  // coupling to the previous row (c | a)
  const int dw = trail ? 1 : -1;
  int off = trail ? 0 : kWin - 1;
  double piv = wB[off];
  double qprev = Qc[off];
  double g = WITH_F ? wF[off] : 0.0;
#pragma unroll
  for (int k = 1; k < kHalo; ++k) {
    off += dw;
    const double l = Nm[off] * fast_rcp(piv);
    piv = fma(-l, qprev, wB[off]);
    qprev = Qc[off];
    if (WITH_F) g = fma(-l, g, wF[off]);
  }
  const double u = fast_rcp(piv);  // v_31 (trailing) or w_0 (leading)
  const double ug = g * u;         // v . f (trailing) or w . f (leading)
  const double ou = __shfl_xor_sync(FULL, u, kFacSeps), oug = __shfl_xor_sync(FULL, ug, kFacSeps);
  if (trail && jj < nj) {
    const double at = wA[kHalo], bt = wB[kHalo], ct = wC[kHalo];  // separator row t
    const double kR = at * wC[kHalo - 1] * u;
    const double kL = ct * wA[kHalo + 1] * ou;
    const double td = b_minus(bt, kR, kL);
    Tdiag[j0 + jj] = td;
    if (WITH_F) xsep[j0 + jj] = ((wF[kHalo] - at * ug) - ct * oug) / td;
  }
  // launched programmatically after the previous solve's certificate kernel:
  // this grid completes only after it (so K3, which waits on this grid, never
  // overwrites the certificate records the previous solve is still reading)
  pdl_wait();
}

// ----------------------------------------------------------------------------
// K3: per-segment solve.  One warp = one segment of <= 32*M body rows; lane t
// owns body rows [tM, tM+M).  M is odd so the stride-M shared-memory walk of
// the warp touches 16 distinct 8-byte bank pairs (2 wavefronts per LDS.64,
// the minimum).  Rows are staged by four lanes issuing one TMA bulk copy each
// (a, b, c, f); x leaves through one TMA bulk store.
//   1. chunk elimination: every chunk row j ends as
//        ap[j] y_first + y_j + cp[j] y_last = dp[j]
//      (row 0: ap y_{prev last} + y_0 + cp y_last; row M-1: ap y_0 + y_{M-1} + cp y_{next first});
//   2. the chunk-last unknowns are eliminated, leaving one tridiagonal row
//      per lane in the chunk-first unknowns, solved by 5 shuffle PCR steps;
//   3. chunk back-substitution.
// ----------------------------------------------------------------------------
struct TriSolveArgs {
  TriRows A;
  RowArr F;
  SegMap S;
  const double* xsep;  // nseg-1 separator values (NULL when nseg == 1)
  double* x;           // output, row r at x[r]
  double4* crec;       // per-segment certificate record (NULL: skip), see tri_cert_kernel
  DevStatus* status;
  int seg0;            // first segment of this launch (the host path solves in row chunks)
  int seg_end;         // persistent launch: segments [seg0 + blockIdx.x, seg_end) with stride gridDim.x
  int body;            // 1: also the componentwise backward error of every body row (K3 <.., BODY = true>)
};

template <int M>
struct TriWarpSmem {
  static constexpr int CAP = 32 * M;   // body rows per segment
  static constexpr int ROW = CAP + 6;  // + both separator rows + staging slack, even
  static constexpr int BYTES = 4 * ROW * 8;
};

// PERSIST: one warp per SM slot loops over segments seg0 + blockIdx.x,
// + gridDim.x, ... with two staging buffers -- the next segment's rows are in
// flight while this one is solved (continuous HBM traffic per warp).
template <int M, bool PERSIST = false, bool BODY = false>
__global__ void __launch_bounds__(32) tri_segment_solve_kernel(TriSolveArgs args) {
  static_assert(M % 2 == 1 && M >= 3, "M must be odd and >= 3");
  constexpr int ROW = TriWarpSmem<M>::ROW;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ double sepv[4];
  const int lane = threadIdx.x;
  const int nseg = args.S.nseg;
  const int seg_begin = args.seg0 + blockIdx.x;
  const int seg_end = PERSIST ? args.seg_end : seg_begin + 1;
  const int stride = PERSIST ? gridDim.x : 1;
  const RowArr X = lane == 0 ? args.A.a : lane == 1 ? args.A.b : lane == 2 ? args.A.c : args.F;
  if (lane == 0) {
    mbar_init(&bars[0], 4);
    if (PERSIST) mbar_init(&bars[1], 4);
  }
  __syncwarp();
  // ---- staging: lanes 0..3 issue one bulk copy each (a, b, c, f rows s-1 .. s+L)
  auto issue = [&](int sg, int buf) -> int {
    long s0;
    int L0;
    seg_of(args.S, sg, s0, L0);
    int sh = 0;
    if (lane < 4) {
      uint32_t tx = 0;
      sh = stage_issue(X, s0 - 1, s0 + L0 + 1, smem + (buf * 4 + (lane & 3)) * ROW, &bars[buf], &tx);
      mbar_arrive_expect_tx(&bars[buf], tx);
    }
    return sh;
  };
  int shift = seg_begin < seg_end ? issue(seg_begin, 0) : 0;
  pdl_wait();     // the separator values come from the previous kernel (staging above overlaps it)
  pdl_trigger();  // the certificate kernel may launch (it waits for this grid before reading the records)
  int k = 0;
  for (int seg = seg_begin; seg < seg_end; seg += stride, ++k) {
  const int buf = PERSIST ? (k & 1) : 0;
  const int shift_next = (PERSIST && seg + stride < seg_end) ? issue(seg + stride, buf ^ 1) : 0;
  long s;
  int L;
  seg_of(args.S, seg, s, L);
  const bool has_l = seg > 0, has_r = seg < nseg - 1;
  const long lo = s - 1, hi = s + L + 1;
  double* const base = smem + (buf * 4 + (lane & 3)) * ROW;
  // sX[q] = body row q; sX[-1] / sX[L] = left / right separator rows
  double* sA = smem + (buf * 4 + 0) * ROW + 2 + __shfl_sync(FULL, shift, 0);
  double* sB = smem + (buf * 4 + 1) * ROW + 2 + __shfl_sync(FULL, shift, 1);
  double* sC = smem + (buf * 4 + 2) * ROW + 2 + __shfl_sync(FULL, shift, 2);
  double* sF = smem + (buf * 4 + 3) * ROW + 2 + __shfl_sync(FULL, shift, 3);
  const double xl = has_l ? args.xsep[seg - 1] : 0.0;
  const double xr = has_r ? args.xsep[seg] : 0.0;
  mbar_wait(&bars[buf], PERSIST ? ((k >> 1) & 1) : 0);
  if (lane < 4) stage_fixup(X, lo, hi, base + 1 + shift);
  __syncwarp();
  if (lane == 0) {
    sepv[0] = sA[L];  // separator-row entries for the certificate record
    sepv[1] = sB[L];
    sepv[2] = sF[L];
    sepv[3] = sC[-1];
    sF[0] = fma(-sA[0], xl, sF[0]);  // fold the separator couplings into the rhs
    sA[0] = 0.0;
    sF[L - 1] = fma(-sC[L - 1], xr, sF[L - 1]);
    sC[L - 1] = 0.0;
  }
  for (int q = L + lane; q < 32 * M; q += 32) {  // decoupled identity padding
    sA[q] = 0.0;
    sB[q] = 1.0;
    sC[q] = 0.0;
    sF[q] = 0.0;
  }
  __syncwarp();

  // ---- chunk elimination: every chunk row j ends as
  //      ap[j] y_first + y_j + cp[j] y_last = dp[j]
  //      (row 0: ap y_{prev last} + y_0 + cp y_last; row M-1: ap y_0 + y_{M-1} + cp y_{next first})
  double ap[M], cp[M], dp[M];
  const int q0 = lane * M;
  double rsum = 0.0;  // sum of |pivot reciprocals|: non-finite <=> a pivot of this body vanished
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const double a = sA[q0 + j], b = sB[q0 + j], c = sC[q0 + j], f = sF[q0 + j];
    double r;
    if (j < 2) {
      r = fast_rcp(b);
      ap[j] = a * r;
      cp[j] = c * r;
      dp[j] = f * r;
    } else {
      r = fast_rcp(fma(-a, cp[j - 1], b));
      dp[j] = r * fma(-a, dp[j - 1], f);
      ap[j] = -r * a * ap[j - 1];
      cp[j] = r * c;
    }
    rsum += fabs(r);
  }
#pragma unroll
  for (int j = M - 3; j >= 1; --j) {
    dp[j] = fma(-cp[j], dp[j + 1], dp[j]);
    ap[j] = fma(-cp[j], ap[j + 1], ap[j]);
    cp[j] = -cp[j] * cp[j + 1];
  }
  {
    const double r = fast_rcp(fma(-cp[0], ap[1], 1.0));
    rsum += fabs(r);
    dp[0] = r * fma(-cp[0], dp[1], dp[0]);
    ap[0] = r * ap[0];
    cp[0] = -r * cp[0] * cp[1];
  }

  // ---- chunk interfaces -> one normalised tridiagonal row per lane in F = y_first
  const double aE = ap[M - 1], cE = cp[M - 1], dE = dp[M - 1];
  double pa = __shfl_up_sync(FULL, aE, 1), pc = __shfl_up_sync(FULL, cE, 1), pd = __shfl_up_sync(FULL, dE, 1);
  if (lane == 0) pa = pc = pd = 0.0;
  double al = -ap[0] * pa;
  double ga = -cp[0] * cE;
  double de = dp[0] - ap[0] * pd - cp[0] * dE;
  {
    const double r = fast_rcp(1.0 - ap[0] * pc - cp[0] * aE);
    rsum += fabs(r);
    al *= r;
    ga *= r;
    de *= r;
  }
#pragma unroll
  for (int st = 1; st < 32; st <<= 1) {
    double la = __shfl_up_sync(FULL, al, st), lg = __shfl_up_sync(FULL, ga, st), ld = __shfl_up_sync(FULL, de, st);
    double ha = __shfl_down_sync(FULL, al, st), hg = __shfl_down_sync(FULL, ga, st),
           hd = __shfl_down_sync(FULL, de, st);
    if (lane < st) la = lg = ld = 0.0;
    if (lane + st >= 32) ha = hg = hd = 0.0;
    const double r = fast_rcp(1.0 - al * lg - ga * ha);
    rsum += fabs(r);
    const double nde = de - al * ld - ga * hd;
    al = -al * la * r;
    ga = -ga * hg * r;
    de = nde * r;
  }
  const double Fv = de;
  double Fn = __shfl_down_sync(FULL, Fv, 1);
  if (lane == 31) Fn = 0.0;
  const double Ev = dE - aE * Fv - cE * Fn;

  // ---- chunk back-substitution, finite check, stage y over f.  BODY: the
  // componentwise backward error of every body row too (the row's f is read
  // before y overwrites it; separator couplings are folded into f, which only
  // shrinks the denominator: a conservative bound), no extra HBM traffic.
  bool finite = true;
  double wnum = 0.0, wden = 1.0;  // largest num / den so far, compared by cross products (no division per row)
  double ym2 = BODY ? __shfl_up_sync(FULL, Ev, 1) : 0.0, ym1 = 0.0, fm1 = 0.0;  // y_{q0-1}: previous chunk's last
  if (BODY && lane == 0) ym2 = 0.0;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const double y = (j == 0) ? Fv : (j == M - 1) ? Ev : dp[j] - ap[j] * Fv - cp[j] * Ev;
    if (q0 + j < L) finite &= isfinite(y);
    if (BODY) {
      const double fj = sF[q0 + j];
      if (j > 0) {  // row q0 + j - 1: a y_{j-2} + b y_{j-1} + c y_j = f
        const int q = q0 + j - 1;
        const double ta = sA[q] * ym2, tb = sB[q] * ym1, tc = sC[q] * y;
        const double num = fabs(((fm1 - ta) - tb) - tc), den = fabs(fm1) + fabs(ta) + fabs(tb) + fabs(tc);
        if (q < L && !(num * wden <= wnum * den)) {  // NaN-safe: a non-finite row always wins
          wnum = num;
          wden = den;
        }
      }
      ym2 = j > 0 ? ym1 : ym2;
      ym1 = y;
      fm1 = fj;
    }
    sF[q0 + j] = y;
  }
  if (BODY) {  // the chunk's last row: its right neighbour is the next chunk's first (Fn)
    const int q = q0 + M - 1;
    const double ta = sA[q] * ym2, tb = sB[q] * ym1, tc = sC[q] * Fn;
    const double num = fabs(((fm1 - ta) - tb) - tc), den = fabs(fm1) + fabs(ta) + fabs(tb) + fabs(tc);
    if (q < L && !(num * wden <= wnum * den)) {
      wnum = num;
      wden = den;
    }
    double wbody = wden > 0.0 ? wnum / wden : (wnum > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0);
    if (!(wbody <= 1.0e300)) wbody = __longlong_as_double(0x7ff0000000000000ll);
    for (int o = 16; o > 0; o >>= 1) wbody = fmax(wbody, __shfl_xor_sync(FULL, wbody, o));
    if (lane == 0 && wbody > 0.0 && args.status) status_cert(args.status, wbody);
  }
  if (args.status) {
    const bool piv_ok = __all_sync(FULL, isfinite(rsum));
    const bool all_ok = __all_sync(FULL, finite);
    if (lane == 0) {
      if (!piv_ok) status_pivot(args.status, seg);
      if (!all_ok) status_nonfinite(args.status, seg);
    }
  }
  fence_proxy_async_smem();
  __syncwarp();

  // ---- write-back: aligned interior by one TMA bulk store, ragged ends by lanes 1/2
  double* xg = args.x + s;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(xg), a1 = reinterpret_cast<uintptr_t>(xg + L);
  const uintptr_t b0 = (a0 + 15) & ~uintptr_t(15), b1 = a1 & ~uintptr_t(15);
  const bool congruent = ((a0 - reinterpret_cast<uintptr_t>(sF)) & 15) == 0;
  if (congruent && b1 > b0) {
    if (lane == 0) {
      bulk_s2g(reinterpret_cast<void*>(b0), sF + ((b0 - a0) >> 3), (uint32_t)(b1 - b0));
      bulk_commit_and_wait_read();
    }
    if (lane == 1 && a0 < b0) xg[0] = sF[0];
    if (lane == 2 && a1 > b1) xg[L - 1] = sF[L - 1];
  } else {
    for (int q = lane; q < L; q += 32) xg[q] = sF[q];
  }
  if (lane == 3) {
    if (has_r) args.x[s + L] = xr;
    // certificate record: right separator t = s+L: (a_t y_{t-1}, b_t x_t, f_t),
    // left separator: c_{s-1} y_s
    if (args.crec) {
      args.crec[seg] = make_double4(has_r ? sepv[0] * sF[L - 1] : 0.0, has_r ? sepv[1] * xr : 0.0,
                                    has_r ? sepv[2] : 0.0, has_l ? sepv[3] * sF[0] : 0.0);
    }
  }
  if (PERSIST) {  // this buffer is refilled by the next iteration's prefetch
    fence_proxy_async_smem();
    __syncwarp();
  }
  shift = shift_next;
  }
}

// ----------------------------------------------------------------------------
// Certificate: componentwise backward error of every separator row,
//   w_t = |f_t - a_t y_{t-1} - b_t x_t - c_t y_{t+1}| / (|f_t| + |a_t y_{t-1}| + |b_t x_t| + |c_t y_{t+1}|)
// with the body values y from K3.  The body rows are solved exactly given
// the separators, so this bounds the error the speculative interface let in.
// ----------------------------------------------------------------------------
// omega of separator j from the records of its two segments (R = j, N = j + 1)
__device__ __forceinline__ double tri_omega(const double4& R, const double4& N) {
  const double r = ((R.z - R.x) - R.y) - N.w;  // f_t - a_t y_{t-1} - b_t x_t - c_t y_{t+1}
  const double den = fabs(R.z) + fabs(R.x) + fabs(R.y) + fabs(N.w);
  double w = den > 0.0 ? fabs(r) / den : (r != 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0);
  if (!(w <= 1.0e300)) w = __longlong_as_double(0x7ff0000000000000ll);
  return w;
}

__global__ void tri_cert_kernel(int nsep, const double4* __restrict__ crec, DevStatus* st, DevStatus* host_out,
                                unsigned* done_ctr) {
  pdl_trigger();  // the next solve's separator kernel may start: it touches nothing K3 or this kernel
                  // reads or writes (other separator buffer, other status slot) and completes only after us
  pdl_wait();     // K3 (records) complete
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double w = 0.0;
  if (j < nsep) w = tri_omega(crec[j], crec[j + 1]);
  for (int o = 16; o > 0; o >>= 1) w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
  if ((threadIdx.x & 31) == 0 && w > 0.0) status_cert(st, w);
  if (host_out) status_publish_last(st, host_out, done_ctr);
}

}  // namespace psg
