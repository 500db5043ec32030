// band_kernels.cuh -- the speculative partition method for Banded matrices
// with s, r <= K (K = separator size = max(s, r), 2..4) worked in SCALAR band
// arithmetic (config 3: s = r = 3).  Same design as blk_kernels.cuh (the K x K
// block view of a band), without the block algebra: a band row has 2K + 1
// entries, the block view's 3 K x K blocks per K rows are 3K entries per row,
// most of them structural zeros, and every block product / inverse ran over
// them.
//
//   separators (band_spec_kernel, lazy factor + condense, one launch per
//     refactor + solve): ONE THREAD PER SEPARATOR SIDE.  The trailing W rows
//     of the body above a separator are eliminated top-down (no-pivot band
//     LU, the reference's banded_factor order, src/localfact.cpp:84-100)
//     carrying f; the last K rows, back-substituted, give the body's near
//     rows as x_near = c + Q x_S (the last K rows of B^-1 [f | C]: the
//     reference's v / y fill-ins restricted to the window, :202-205).  The
//     leading W rows of the body below are eliminated bottom-up (mirror
//     image).  The separator's Schur complement and condensed rhs follow
//     (src/localfact.cpp:207-210, 765-781 on the truncated bodies):
//       (A_SS - A_SL Q_top - A_SR Q_bot) x_S = f_S - A_SL c_top - A_SR c_bot.
//     The windows arrive by warp-cooperative 16-byte cp.async pieces into a
//     per-thread region; 2K + 2 loads of the thread's own rows per step.
//   bodies (band_body_kernel): warp per body, exact given the separators.
//     Lane t owns a chunk of about L / 32 rows: its first K rows are a
//     lane-level separator S_t (lane 0: the body's left separator, known),
//     the rest its sub-body.  Per lane: a forward band-LU sweep carrying
//     [f | spike of S_t] (the stored U rows and condensed rhs replace the
//     staged rows in place), a backward sweep leaving every sub-body row as
//     an affine form x = c + P X_{S_t} + Q X_{S_{t+1}} (2K + 1 values, in
//     place again), the lane-level reduced system (K x K block tridiagonal,
//     one block row per lane, from the neighbours' forms), block PCR across
//     the lanes, and x = c + P X_t + Q X_{t+1}.  One TMA bulk store of x.
//   certificate: blk_cert_kernel (same records as the block body kernels).
#pragma once

#include "blk_kernels.cuh"

namespace psg {

// K x K inverse with a short dependency chain: cofactors / determinant for
// K = 2, 3 (one reciprocal), Gauss-Jordan otherwise.  Used on the lane-level
// reduced rows, which are block diagonally dominant (near-identity after the
// first normalisation).  |1/det| (or the pivot reciprocals) -> *rsum.
template <int K>
__device__ __forceinline__ void blk_inv_short(Blk<K>& A, double* rsum) {
  if constexpr (K == 3) {
    const double a00 = A.v[0][0], a01 = A.v[0][1], a02 = A.v[0][2];
    const double a10 = A.v[1][0], a11 = A.v[1][1], a12 = A.v[1][2];
    const double a20 = A.v[2][0], a21 = A.v[2][1], a22 = A.v[2][2];
    const double c00 = fma(a11, a22, -a12 * a21), c01 = fma(a12, a20, -a10 * a22), c02 = fma(a10, a21, -a11 * a20);
    const double r = fast_rcp(fma(a00, c00, fma(a01, c01, a02 * c02)));
    *rsum += fabs(r);
    A.v[0][0] = c00 * r;
    A.v[1][0] = c01 * r;
    A.v[2][0] = c02 * r;
    A.v[0][1] = fma(a02, a21, -a01 * a22) * r;
    A.v[0][2] = fma(a01, a12, -a02 * a11) * r;
    A.v[1][1] = fma(a00, a22, -a02 * a20) * r;
    A.v[1][2] = fma(a02, a10, -a00 * a12) * r;
    A.v[2][1] = fma(a01, a20, -a00 * a21) * r;
    A.v[2][2] = fma(a00, a11, -a01 * a10) * r;
  } else if constexpr (K == 2) {
    const double r = fast_rcp(fma(A.v[0][0], A.v[1][1], -A.v[0][1] * A.v[1][0]));
    *rsum += fabs(r);
    const double a00 = A.v[0][0];
    A.v[0][0] = A.v[1][1] * r;
    A.v[1][1] = a00 * r;
    A.v[0][1] = -A.v[0][1] * r;
    A.v[1][0] = -A.v[1][0] * r;
  } else {
    blk_inv<K>(A, rsum);
  }
}

template <int K>
__device__ __forceinline__ double blk_maxabs(const Blk<K>& A) {
  double m = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) m = fmax(m, fabs(A.v[i][j]));
  return m;
}

// ---------------------------------------------------------------------------
// bodies
// ---------------------------------------------------------------------------
// smem: 2K + 2 arrays (bands d = -K..K, then f / x) of RB doubles each, RB even
// and >= maxL + 3.  Array a holds body row i at sm[bo[a] + i].
template <int K>
__global__ void __launch_bounds__(32) band_body_kernel(BlkArgs g, int RB) {
  constexpr int E = 2 * K + 1;  // band arrays, a = d + K
  constexpr int NA = E + 1;     // + f (becomes x)
  constexpr int FA = E;
  constexpr int C = 2 * K + 1;  // affine form [const | P (K) | Q (K)]
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int boffs[NA];
  const int lane = threadIdx.x;
  const int seg = blockIdx.x;
  const GPart Pt = g.part[seg];
  const long b = Pt.b;
  const int L = Pt.L;
  const long n = g.n;

  // ---- staging: one TMA bulk copy per band and for f (rows [b, b + L))
  if (lane == 0) mbar_init(&bar, NA);
  __syncwarp();
  RowArr X{};
  if (lane < NA) {
    if (lane == FA) {
      X = make_rows(g.f, 0, (int)n, 0, n);
    } else {
      const int d = lane - K;
      const bool inb = d >= -g.s && d <= g.r;
      const long bo = inb ? g.boff[lane] : 0;
      X = make_rows(g.data + bo, inb ? (d < 0 ? -d : 0) : 0, inb ? (int)(n - (d > 0 ? d : 0)) : 0, -bo,
                    g.data_len - bo);
    }
    uint32_t tx = 0;
    const int shift = stage_issue(X, b, b + L, sm + lane * RB, &bar, &tx);
    mbar_arrive_expect_tx(&bar, tx);
    boffs[lane] = lane * RB + 1 + shift;
  }
  // certificate couplings, loaded while the rows stage: lanes u < K: A(ls + u, b + t),
  // lanes 16 + u: A(rs + u, b + L - 1 - t), t < K (blk_cert_kernel record format)
  double cpl[K];
  {
    const bool left = lane < K, right = lane >= 16 && lane < 16 + K;
    const int u = left ? lane : lane - 16;
    const long row = left ? (long)Pt.ls + u : (long)Pt.rs + u;
    const bool has = (left && Pt.ls >= 0) || (right && Pt.rs >= 0);
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const long col = left ? b + t : b + L - 1 - t;
      const int d = (int)(col - row);
      cpl[t] = (has && g.rec && t < L && d >= -g.s && d <= g.r) ? __ldg(g.data + g.boff[d + K] + row) : 0.0;
    }
  }
  Vec<K> xl, xrv;
  pdl_wait();     // separator values from the separator kernel (the staging above overlaps it)
  pdl_trigger();  // the certificate kernel may launch (it waits for this grid before reading the records)
#pragma unroll
  for (int u = 0; u < K; ++u) {
    xl.v[u] = Pt.ls >= 0 ? __ldg(g.xsep + (long)(seg - 1) * K + u) : 0.0;
    xrv.v[u] = Pt.rs >= 0 ? __ldg(g.xsep + (long)seg * K + u) : 0.0;
  }
  mbar_wait(&bar, 0);
  if (lane < NA) stage_fixup(X, b, b + L, sm + boffs[lane]);
  __syncwarp();
  int bo[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) bo[a] = boffs[a];
  auto S = [&](int a, int i) -> double& { return sm[bo[a] + i]; };

  // ---- lane chunks: lane t's sub-body is [t R, (t + 1) R - K) (the last lane: up to L),
  //      its separator S_t the K rows before it (lane 0: the body's left
  //      separator, known); R odd, so the lanes' rows at the same step fall in
  //      distinct shared-memory banks
  int R = ((L + 31) / 32) | 1;
  if (R < 2 * K) R = (2 * K) | 1;
  int NL = (L + R - 1) / R;
  if (NL > 1 && L - (NL - 1) * R < K) --NL;  // too short a tail: the previous lane takes it
  const bool act = lane < NL;
  const int bl = act ? lane * R : L;                          // sub-body start
  const int hi = act ? (lane + 1 == NL ? L : (lane + 1) * R - K) : L;
  const int sS = bl - K;                                      // S_t start (lane 0: -K, the left separator)
  double rsum = 0.0;

  // ---- forward sweep: no-pivot band LU carrying v = [f | spike of S_t]; the
  //      eliminated row is stored NORMALISED (divided by its pivot: no
  //      reciprocal to keep) in place of its staged entries: super slots
  //      u'_i,i+k, sub slots spike', f slot g'.  7 values per row (K = 3).
  {
    double wu[K][K], wv[K][K + 1];  // window of normalised rows: [0] = row i-1, ..., [K-1] = row i-K
#pragma unroll
    for (int w = 0; w < K; ++w) {
#pragma unroll
      for (int k = 0; k < K; ++k) wu[w][k] = 0.0;
#pragma unroll
      for (int q = 0; q <= K; ++q) wv[w][q] = 0.0;
    }
    // in[]: row i's staged entries (bands, then f), loaded one row ahead
    auto step = [&](int i, int mpeel, const double (&in)[NA]) {  // mpeel: sub-body row when < K, else -1
      double e[E], v[K + 1];
#pragma unroll
      for (int a = 0; a < E; ++a) e[a] = in[a];
      v[0] = in[FA];
#pragma unroll
      for (int q = 1; q <= K; ++q) v[q] = 0.0;
      if (mpeel >= 0) {
#pragma unroll
        for (int c = -K; c < 0; ++c)
          if (mpeel + c < 0) {  // column i + c lies in S_t (index mpeel + K + c): to the rhs
            v[1 + mpeel + K + c] = -e[c + K];
            e[c + K] = 0.0;
          }
      }
#pragma unroll
      for (int c = -K; c < 0; ++c) {  // the multiplier is the entry itself (rows normalised)
        const int w = -c - 1;
        const double l = e[c + K];
#pragma unroll
        for (int k = 1; k <= K; ++k)
          if (c + k <= K) e[c + k + K] = fma(-l, wu[w][k - 1], e[c + k + K]);
#pragma unroll
        for (int q = 0; q <= K; ++q) v[q] = fma(-l, wv[w][q], v[q]);
      }
      const double r = fast_rcp(e[K]);
      rsum += fabs(r);
#pragma unroll
      for (int w = K - 1; w > 0; --w) {
#pragma unroll
        for (int k = 0; k < K; ++k) wu[w][k] = wu[w - 1][k];
#pragma unroll
        for (int q = 0; q <= K; ++q) wv[w][q] = wv[w - 1][q];
      }
#pragma unroll
      for (int k = 0; k < K; ++k) wu[0][k] = e[K + 1 + k] * r;
#pragma unroll
      for (int q = 0; q <= K; ++q) wv[0][q] = v[q] * r;
#pragma unroll
      for (int k = 1; k <= K; ++k) S(K + k, i) = wu[0][k - 1];
#pragma unroll
      for (int q = 1; q <= K; ++q) S(q - 1, i) = wv[0][q];
      S(FA, i) = wv[0][0];
    };
    if (act) {
      double cur[NA], nxt[NA];
#pragma unroll
      for (int a = 0; a < NA; ++a) cur[a] = S(a, bl);
#pragma unroll
      for (int m = 0; m < K; ++m) {
#pragma unroll
        for (int a = 0; a < NA; ++a) nxt[a] = S(a, bl + m + 1);
        step(bl + m, m, cur);
#pragma unroll
        for (int a = 0; a < NA; ++a) cur[a] = nxt[a];
      }
#pragma unroll (K)
      for (int i = bl + K; i < hi; ++i) {  // row hi is read ahead (inside the region; unused); unrolled by K: the window rotates by renaming
#pragma unroll
        for (int a = 0; a < NA; ++a) nxt[a] = S(a, i + 1);
        step(i, -1, cur);
#pragma unroll
        for (int a = 0; a < NA; ++a) cur[a] = nxt[a];
      }
    }
  }
  // normalised row i: u' (K), then [g' | spike' (K)]
  auto ldrow = [&](double (&f)[2 * K + 1], int i) {
#pragma unroll
    for (int k = 1; k <= K; ++k) f[k - 1] = S(K + k, i);
    f[K] = S(FA, i);
#pragma unroll
    for (int q = 1; q <= K; ++q) f[K + q] = S(q - 1, i);
  };
  // ---- backward sweep 1, in registers only: the affine forms
  //      x_i = c + P X_{S_t} + Q X_{S_{t+1}} of the rows the lane-level reduced
  //      system needs -- the K lowest (bot[m] = row hi-1-m, from the first K
  //      steps) and the K highest (wx[w] = row bl + w, what the window holds at
  //      the end).  Nothing is stored: backward sweep 2 recomputes x from the
  //      normalised rows once X is known (7 loads and 1 store per row instead
  //      of 7 stores and 7 loads of forms).
  double wx[K][C], bot[K][C];  // wx: [0] = row i+1, ...
  if (act) {
    auto step = [&](int mpeel, const double (&in)[2 * K + 1]) {  // mpeel: rows below i in the sub-body when < K
      double x[C];
      x[0] = in[K];
#pragma unroll
      for (int q = 1; q <= K; ++q) x[q] = in[K + q];
#pragma unroll
      for (int q = K + 1; q < C; ++q) x[q] = 0.0;
#pragma unroll
      for (int k = 1; k <= K; ++k) {
        const double u = in[k - 1];
        if (mpeel < 0 || k <= mpeel) {
#pragma unroll
          for (int q = 0; q < C; ++q) x[q] = fma(-u, wx[k - 1][q], x[q]);
        } else {  // row i + k = hi + (k - 1 - mpeel): row k - 1 - mpeel of S_{t+1}
          x[K + 1 + (k - 1 - mpeel)] -= u;
        }
      }
#pragma unroll
      for (int w = K - 1; w > 0; --w)
#pragma unroll
        for (int q = 0; q < C; ++q) wx[w][q] = wx[w - 1][q];
#pragma unroll
      for (int q = 0; q < C; ++q) wx[0][q] = x[q];
    };
    double cur[2 * K + 1], nxt[2 * K + 1];
    ldrow(cur, hi - 1);
#pragma unroll
    for (int m = 0; m < K; ++m) {
      ldrow(nxt, hi - 2 - m);
      step(m, cur);
#pragma unroll
      for (int q = 0; q < C; ++q) bot[m][q] = wx[0][q];
#pragma unroll
      for (int a = 0; a < 2 * K + 1; ++a) cur[a] = nxt[a];
    }
#pragma unroll (K)
    for (int i = hi - 1 - K; i >= bl; --i) {  // row bl - 1 is read ahead (inside the region; unused); unrolled by K
      ldrow(nxt, i - 1);
      step(-1, cur);
#pragma unroll
      for (int a = 0; a < 2 * K + 1; ++a) cur[a] = nxt[a];
    }
  } else {
#pragma unroll
    for (int w = 0; w < K; ++w)
#pragma unroll
      for (int q = 0; q < C; ++q) wx[w][q] = bot[w][q] = 0.0;
  }
  // the previous lane's lowest forms (rows sS-1-m)
  double pbot[K][C];
#pragma unroll
  for (int m = 0; m < K; ++m)
#pragma unroll
    for (int q = 0; q < C; ++q) pbot[m][q] = __shfl_sync(FULL, bot[m][q], lane > 0 ? lane - 1 : 0);

  // ---- lane-level reduced system: the K rows of S_t,
  //      Ab X_{S_{t-1}} + Bb X_{S_t} + Cb X_{S_{t+1}} = Fv
  Blk<K> Ab, Bb, Cb;
  Vec<K> Fv;
  blk_set_zero<K>(Ab);
  blk_set_zero<K>(Cb);
  blk_set_eye<K>(Bb);
#pragma unroll
  for (int u = 0; u < K; ++u) Fv.v[u] = 0.0;
  if (lane == 0) {
    Fv = xl;
  } else if (act) {
    blk_set_zero<K>(Bb);
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const int rho = sS + u;
      double fv = S(FA, rho);
#pragma unroll
      for (int c = -K; c <= K; ++c) {
        const double a = S(c + K, rho);
        if (u + c >= 0 && u + c < K) {
          Bb.v[u][u + c] += a;
        } else {  // a sub-body row: the previous lane's (P: S_{t-1}, Q: S_t) or ours (P: S_t, Q: S_{t+1})
          const bool prev = u + c < 0;
          const double* fm = prev ? pbot[-(u + c) - 1] : wx[u + c - K];  // compile-time indices
          fv = fma(-a, fm[0], fv);
#pragma unroll
          for (int v = 0; v < K; ++v) {
            const double P = fm[1 + v], Q = fm[1 + K + v];
            if (prev) {
              Ab.v[u][v] = fma(a, P, Ab.v[u][v]);
              Bb.v[u][v] = fma(a, Q, Bb.v[u][v]);
            } else {
              Bb.v[u][v] = fma(a, P, Bb.v[u][v]);
              Cb.v[u][v] = fma(a, Q, Cb.v[u][v]);
            }
          }
        }
      }
      Fv.v[u] = fv;
    }
    if (lane == NL - 1) {  // S_{t+1} is the body's right separator (known)
      blk_mv_sub<K>(Fv, Cb, xrv);
      blk_set_zero<K>(Cb);
    }
  }
  // ---- normalise and solve the lane-level system (al = B^-1 A, ga = B^-1 C,
  //      de = B^-1 F).  It is block diagonally dominant for the bodies this
  //      path certifies: strongly decoupled rows take block Jacobi sweeps
  //      (blk_jacobi: config 3 kappa ~ 1e-7, 2 sweeps), otherwise block PCR,
  //      left once every coupling is below 2^-64 (X changes by < 1e-19 relative).
  blk_inv_short<K>(Bb, &rsum);
  Blk<K> al = blk_mul<K>(Bb, Ab), ga = blk_mul<K>(Bb, Cb);
  Vec<K> de = blk_mv<K>(Bb, Fv);
  constexpr double kDecoupled = 5.421010862427522e-20;  // 2^-64
  const bool jacobi = blk_jacobi<K>(al, ga, de, lane, 32);
#pragma unroll 1
  for (int st = 1; st < (jacobi ? 1 : NL); st <<= 1) {
    if (__all_sync(FULL, fmax(blk_maxabs<K>(al), blk_maxabs<K>(ga)) < kDecoupled)) break;
    const bool hl = lane >= st, hh = lane + st < 32;
    const int sl = hl ? lane - st : lane, sh = hh ? lane + st : lane;
    Blk<K> nb, na, ng;
    blk_set_eye<K>(nb);
    Vec<K> nd = de;
    {
      const Blk<K> lg = blk_shfl<K>(ga, sl);
      if (hl) blk_mul_sub<K>(nb, al, lg);
      const Blk<K> la = blk_shfl<K>(al, sl);
      if (hl)
        na = blk_mul<K>(al, la);
      else
        blk_set_zero<K>(na);
      const Vec<K> ld = vec_shfl<K>(de, sl);
      if (hl) blk_mv_sub<K>(nd, al, ld);
    }
    {
      const Blk<K> ha = blk_shfl<K>(al, sh);
      if (hh) blk_mul_sub<K>(nb, ga, ha);
      const Blk<K> hg = blk_shfl<K>(ga, sh);
      if (hh)
        ng = blk_mul<K>(ga, hg);
      else
        blk_set_zero<K>(ng);
      const Vec<K> hd = vec_shfl<K>(de, sh);
      if (hh) blk_mv_sub<K>(nd, ga, hd);
    }
    blk_inv_short<K>(nb, &rsum);
    al = blk_mul<K>(nb, na);
    blk_neg<K>(al);
    ga = blk_mul<K>(nb, ng);
    blk_neg<K>(ga);
    de = blk_mv<K>(nb, nd);
  }
  // ---- backward sweep 2: x_i = g'_i + spike'_i . X_t - sum_k u'_ik x_{i+k}
  //      (x_{i+k} of rows >= hi: X_{t+1}) over the sub-body, in place of g';
  //      the S_t rows get X_t
  Vec<K> Xn = vec_shfl<K>(de, lane < 31 ? lane + 1 : lane);
  if (lane == NL - 1) Xn = xrv;
  bool finite = true;
  if (act) {
    double xw[K];  // [0] = x_{i+1}, ...
#pragma unroll
    for (int k = 0; k < K; ++k) xw[k] = Xn.v[k];  // rows hi.. hi+K-1 (for the last rows of the sub-body)
    // the window starts at row hi: x_{hi + k} = Xn[k]; shift it so that xw[k] = x_{i+1+k}
    double cur[2 * K + 1], nxt[2 * K + 1];
    ldrow(cur, hi - 1);
    auto step = [&](int i, const double (&in)[2 * K + 1]) {
      double x = in[K];
#pragma unroll
      for (int q = 0; q < K; ++q) x = fma(in[K + 1 + q], de.v[q], x);
#pragma unroll
      for (int k = K; k >= 1; --k) x = fma(-in[k - 1], xw[k - 1], x);  // x_{i+1} last: shortest chain
      finite &= isfinite(x);
      S(FA, i) = x;
#pragma unroll
      for (int k = K - 1; k > 0; --k) xw[k] = xw[k - 1];
      xw[0] = x;
    };
#pragma unroll (K)
    for (int i = hi - 1; i >= bl; --i) {
      ldrow(nxt, i - 1);
      step(i, cur);
#pragma unroll
      for (int a = 0; a < 2 * K + 1; ++a) cur[a] = nxt[a];
    }
    if (lane > 0)
#pragma unroll
      for (int u = 0; u < K; ++u) {
        finite &= isfinite(de.v[u]);
        S(FA, sS + u) = de.v[u];
      }
  }
  if (g.status) {
    const bool piv_ok = __all_sync(FULL, isfinite(rsum));
    const bool all_ok = __all_sync(FULL, finite);
    if (lane == 0) {
      if (!piv_ok) status_pivot(g.status, seg);
      if (!all_ok) status_nonfinite(g.status, seg);
    }
  }
  fence_proxy_async_smem();
  __syncwarp();
  // ---- write-back: aligned interior by one TMA bulk store, ragged ends by lanes 1/2
  const double* sx = sm + bo[FA];
  {
    double* xg = g.x + b;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(xg), a1 = reinterpret_cast<uintptr_t>(xg + L);
    const uintptr_t b0 = (a0 + 15) & ~uintptr_t(15), b1 = a1 & ~uintptr_t(15);
    const bool congruent = ((a0 - reinterpret_cast<uintptr_t>(sx)) & 15) == 0;
    if (congruent && b1 > b0) {
      if (lane == 0) {
        bulk_s2g(reinterpret_cast<void*>(b0), sx + ((b0 - a0) >> 3), (uint32_t)(b1 - b0));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (lane == 1 && a0 < b0) xg[0] = sx[0];
      if (lane == 2 && a1 > b1) xg[L - 1] = sx[L - 1];
    } else {
      for (int q = lane; q < L; q += 32) xg[q] = sx[q];
    }
  }
  if (lane == 0 && Pt.rs >= 0)
#pragma unroll
    for (int u = 0; u < K; ++u) g.x[Pt.rs + u] = xrv.v[u];
  // ---- certificate records: the separator rows' couplings to this body (blk_cert_kernel format)
  if (g.rec && (lane < K || (lane >= 16 && lane < 16 + K))) {
    const bool left = lane < K;
    const int u = left ? lane : lane - 16;
    double sg = 0.0, ab = 0.0;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const double pr = t < L ? cpl[t] * sx[left ? t : L - 1 - t] : 0.0;
      sg += pr;
      ab += fabs(pr);
    }
    double* rc = g.rec + (long)seg * 4 * K + (left ? 0 : 2 * K);
    rc[u] = sg;
    rc[K + u] = ab;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// separators: thread per separator side
// ---------------------------------------------------------------------------
// rows of array a (bands d = a - K, then f) with a defined value
__device__ __forceinline__ void band_rows(const BlkSpecArgs& g, int K, int a, long& lo, long& hi) {
  if (a == 2 * K + 1) {
    lo = 0;
    hi = g.n;
    return;
  }
  const int d = a - K;
  if (d < -g.s || d > g.r) {
    lo = hi = 0;
    return;
  }
  lo = d < 0 ? -d : 0;
  hi = g.n - (d > 0 ? d : 0);
}

// 32-byte aligned load of 4 doubles (LDG.256, L1 not allocated: the sector
// is used by this thread only, within the next four steps); predicated off:
// zeros
__device__ __forceinline__ void ldg256_or0(const double* p, bool on, double (&v)[4]) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "mov.f64 %0, 0d0000000000000000;\n\tmov.f64 %1, 0d0000000000000000;\n\t"
      "mov.f64 %2, 0d0000000000000000;\n\tmov.f64 %3, 0d0000000000000000;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];\n\t}"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
      : "l"(p), "r"((int)on));
}

constexpr int kBandSpecThreads = 64;  // 32 separators per CTA: warp 0 the sides above, warp 1 below

// One side of a separator, one thread: the W window rows of the body above
// (H = 0: rows S-W..S-1, eliminated top-down) or below (H = 1: rows
// S+K..S+K+W-1, eliminated bottom-up), streamed straight from HBM with no
// shared memory: two rows of every band per 16-byte load, one group of two
// rows ahead of the sweep (occupancy is register-bound).  Window rows in
// memory order [r0, r0 + W); group G = rows [2G, 2G + 2) = elements
// [2G + o, 2G + o + 2) of the aligned pairs from p + r0 - o: pairs G and
// G + 1.  Returns this side's contribution to the separator rows: Ts (added
// to A_SS) and rs (subtracted from f_S).  (Staging the 400-byte windows in
// shared memory -- TMA bulk copies or cp.async -- held the kernel at 2 warps
// per SM: 128-181 us at config 3.)
template <int K, int W, int H>
__device__ __forceinline__ bool band_side(const BlkSpecArgs& g, bool live, long Ssep, double (&Ts)[K][K],
                                          double (&rs)[K]) {
  constexpr int E = 2 * K + 1, NA = E + 1, FA = E;
  constexpr int NG = W / 4;
  static_assert(W % 4 == 0, "window rows: a multiple of 4");
  const long n = g.n;
  const long r0 = H == 0 ? Ssep - W : Ssep + K;
  // sweep entry c (offset c - K; entry E: f) -> array a: band c top-down, 2K - c bottom-up
  auto arr_of = [&](int c) { return c == E ? FA : (H == 0 ? c : 2 * K - c); };
  auto ptr = [&](int c) -> const double* { return c == E ? g.f : g.data + g.boff[arr_of(c)]; };
  unsigned offm = 0, on = 0;  // 2 bits per entry: element of row r0 in its block; bit: entry loaded
  bool plain = live;          // every window row defined, the blocks inside the allocation
#pragma unroll
  for (int c = 0; c <= E; ++c) {
    const int a = arr_of(c);
    if (a != FA && (a - K < -g.s || a - K > g.r)) continue;  // band not stored: zeros
    long lo, hi, slo, shi;
    band_rows(g, K, a, lo, hi);
    slo = a == FA ? 0 : -g.boff[a];
    shi = a == FA ? n : g.data_len - g.boff[a];
    const unsigned o = (unsigned)((reinterpret_cast<uintptr_t>(ptr(c) + r0) >> 3) & 3);
    offm |= o << (2 * c);
    on |= 1u << c;
    plain &= r0 - (long)o >= slo && r0 - (long)o + W + 4 <= shi && lo <= r0 && hi >= r0 + W;
  }
  // The host only takes this path for interior windows; a thread whose window
  // is not (plain false) loads nothing and returns NaN, which the certificate rejects.
  if (!plain) on = 0;
  auto ldblk = [&](int c, int b, double (&v)[4]) {
    ldg256_or0(ptr(c) + r0 - (long)((offm >> (2 * c)) & 3) + 4 * b, (on >> c) & 1, v);
  };
  // group G = memory rows [4G, 4G + 4) = elements [4G + o, 4G + o + 4): blocks G and G + 1.
  // pA: the block this group shares with the next one (H = 0: G + 1, H = 1: G); the
  // group's rows are extracted first, then pA moves on and the next new block lands in it.
  double pA[NA][4], pB[NA][4];
  constexpr int G0 = H == 0 ? 0 : NG - 1;
#pragma unroll
  for (int c = 0; c <= E; ++c) {
    ldblk(c, H == 0 ? G0 + 1 : G0, pA[c]);
    ldblk(c, H == 0 ? G0 : G0 + 1, pB[c]);
  }
  double wr[K], wu[K][K], wv[K];  // window: [0] = the row just eliminated, [w] = w rows before
#pragma unroll
  for (int w = 0; w < K; ++w) {
    wr[w] = 0.0;
    wv[w] = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) wu[w][k] = 0.0;
  }
  double rsum = plain ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
#pragma unroll 1
  for (int q = 0; q < NG; ++q) {
    const int G = H == 0 ? q : NG - 1 - q;
    // memory row i of entry c: element i + o of [block G | block G + 1]; into pB
#pragma unroll
    for (int c = 0; c <= E; ++c) {
      double t8[8];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        t8[x] = H == 0 ? pB[c][x] : pA[c][x];
        t8[4 + x] = H == 0 ? pA[c][x] : pB[c][x];
      }
      const unsigned o = (offm >> (2 * c)) & 3;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const double lo = (o & 1) ? t8[x + 1] : t8[x];
        const double hi = (o & 1) ? t8[x + 3] : t8[x + 2];
        pB[c][x] = (o & 2) ? hi : lo;
      }
    }
    double pN[NA][4];
    if (q + 1 < NG) {  // the next group's new block: H = 0: G + 2, H = 1: G - 1
#pragma unroll
      for (int c = 0; c <= E; ++c) ldblk(c, H == 0 ? G + 2 : G - 1, pN[c]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = H == 0 ? t : 3 - t;  // memory row in the group, in sweep order
      double e[E], v;
#pragma unroll
      for (int c = 0; c < E; ++c) e[c] = pB[c][i];
      v = pB[E][i];
#pragma unroll
      for (int c = -K; c < 0; ++c) {
        const int w = -c - 1;
        const double l = e[c + K] * wr[w];
#pragma unroll
        for (int k = 1; k <= K; ++k)
          if (c + k <= K) e[c + k + K] = fma(-l, wu[w][k - 1], e[c + k + K]);
        v = fma(-l, wv[w], v);
      }
      const double r = fast_rcp(e[K]);
      rsum += fabs(r);
#pragma unroll
      for (int w = K - 1; w > 0; --w) {
        wr[w] = wr[w - 1];
        wv[w] = wv[w - 1];
#pragma unroll
        for (int k = 0; k < K; ++k) wu[w][k] = wu[w - 1][k];
      }
      wr[0] = r;
      wv[0] = v;
#pragma unroll
      for (int k = 0; k < K; ++k) wu[0][k] = e[K + 1 + k];
    }
#pragma unroll
    for (int c = 0; c <= E; ++c)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        pB[c][x] = pA[c][x];
        pA[c][x] = pN[c][x];
      }
  }
  if (!plain) wv[0] = rsum;  // NaN separator
  // The window now holds the K rows nearest the separator: [q] at distance
  // q + 1.  Back-substitution: x_near(q) = c_q + sum_v Q_q[v] x_S(v), v the
  // separator row counted from this side's end (step k from distance q + 1
  // reaches distance q + 1 - k; k > q: separator row k - q - 1).
  double cq[K], Qq[K][K];
#pragma unroll
  for (int q = 0; q < K; ++q) {  // nearest row first: it couples only to the separator
    double c = wv[q], Qv[K];
#pragma unroll
    for (int v = 0; v < K; ++v) Qv[v] = 0.0;
#pragma unroll
    for (int k = 1; k <= K; ++k) {
      const double u = wu[q][k - 1];
      if (k <= q) {
        c = fma(-u, cq[q - k], c);
#pragma unroll
        for (int v = 0; v < K; ++v) Qv[v] = fma(-u, Qq[q - k][v], Qv[v]);
      } else {
        Qv[k - q - 1] -= u;
      }
    }
    cq[q] = c * wr[q];
#pragma unroll
    for (int v = 0; v < K; ++v) Qq[q][v] = Qv[v] * wr[q];
  }
  // contribution to the separator rows u (top-down): the near row at distance
  // q + 1 is S-1-q (H = 0) or S+K+q (H = 1); separator row v from this side's
  // end is column v (H = 0) or K-1-v (H = 1) top-down.
  auto at = [&](long row, long col) -> double {
    const long d = col - row;
    if (row < 0 || row >= n || col < 0 || col >= n || d < -g.s || d > g.r) return 0.0;
    return __ldg(g.data + g.boff[d + K] + row);
  };
#pragma unroll
  for (int u = 0; u < K; ++u) {
    rs[u] = 0.0;
#pragma unroll
    for (int v = 0; v < K; ++v) Ts[u][v] = 0.0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const double a = live ? at(Ssep + u, H == 0 ? Ssep - 1 - q : Ssep + K + q) : 0.0;
      rs[u] = fma(a, cq[q], rs[u]);
#pragma unroll
      for (int v = 0; v < K; ++v) {
        const int col = H == 0 ? v : K - 1 - v;
        Ts[u][col] = fma(a, Qq[q][v], Ts[u][col]);
      }
    }
  }
  return isfinite(rsum);
}

// Separator kernel: CTA = 2 warps over 32 separators; warp 0 sweeps the sides
// above, warp 1 the sides below (the side is warp-uniform: no divergence, no
// selects), the lower half of the pair combines through shared memory:
//   (A_SS + Ts_above + Ts_below) x_S = f_S - rs_above - rs_below.
template <int K, int W>
__global__ void __launch_bounds__(kBandSpecThreads) band_spec_kernel(BlkSpecArgs g) {
  __shared__ double xch[32][K * K + K];
  const int tid = threadIdx.x;
  if (g.reset && blockIdx.x == 0)  // first kernel of the solve: fresh status
    for (int q = tid; q < kCertSlots + 2; q += blockDim.x) {
      if (q < kCertSlots)
        g.reset->cert_bits[q] = 0ull;
      else if (q == kCertSlots)
        g.reset->bad_seg = INT_MAX;
      else
        g.reset->pivot_seg = INT_MAX;
    }
  const int lane = tid & 31, h = tid >> 5;
  const int j = blockIdx.x * 32 + lane;
  const bool live = j < g.nsep;
  const long Ssep = live ? g.sep[j] : 0;
  pdl_trigger();  // the body kernel may launch and stage its rows while the sides are swept
  double Ts[K][K], rs[K];
  if (h == 0)
    band_side<K, W, 0>(g, live, Ssep, Ts, rs);
  else
    band_side<K, W, 1>(g, live, Ssep, Ts, rs);
  if (h == 1) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
      xch[lane][K * K + u] = rs[u];
#pragma unroll
      for (int v = 0; v < K; ++v) xch[lane][u * K + v] = Ts[u][v];
    }
  }
  __syncthreads();
  if (h == 0 && live) {
    const long n = g.n;
    auto at = [&](long row, long col) -> double {
      const long d = col - row;
      if (row < 0 || row >= n || col < 0 || col >= n || d < -g.s || d > g.r) return 0.0;
      return __ldg(g.data + g.boff[d + K] + row);
    };
    Blk<K> T;
    Vec<K> rhs;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      rhs.v[u] = (__ldg(g.f + Ssep + u) - rs[u]) - xch[lane][K * K + u];
#pragma unroll
      for (int v = 0; v < K; ++v) {
        const double ass = at(Ssep + u, Ssep + v);
        T.v[u][v] = ass + Ts[u][v] + xch[lane][u * K + v];  // Q carries the minus sign of the substitution
        g.Tdiag[(long)j * K * K + u * K + v] = ass;
      }
    }
    double rsum = 0.0;
    blk_inv<K>(T, &rsum);
    const Vec<K> xs = blk_mv<K>(T, rhs);
#pragma unroll
    for (int u = 0; u < K; ++u) g.xsep[(long)j * K + u] = xs.v[u];
  }
  // a vanished pivot leaves non-finite separator values: the certificate rejects them
}

}  // namespace psg
