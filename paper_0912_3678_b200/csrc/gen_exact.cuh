// gen_exact.cuh -- exact partition method for every structured kind
// (Banded with any s, r; BlockTridiagonal; Abd; Babd with corner), following
// the reference's scalar-envelope elimination (src/localfact.cpp:84-225):
//
//   per partition i (body rows [b, b+L), left/right separators of size k):
//     factor   : alpha1 = -C0 B^-1 B0, alpha2 = a_right - B1 B^-1 C1,
//                beta = -B1 B^-1 B0,   gamma = -C0 B^-1 C1
//     condense : kept_rhs = [-C0 B^-1 f ; -B1 B^-1 f]
//     backsolve: x_body = B^-1 (f - B0 x_left - C1 x_right)
//   with B0/C1 the body->separator columns and C0/B1 the separator->body rows
//   (src/partition.cpp:136-162).
//
// Only the first rows (C0 touches the first er+k body columns) or the last
// rows (B1 touches the last es+k) of B^-1 X are needed by factor/condense, so
// each is ONE windowed no-pivot band elimination: top-down (LU) for the last
// rows, bottom-up (UL == LU of the reversed body) for the first rows; neither
// stores the factors.  One warp runs one sweep: rows stream through a ring of
// es+1+CH rows in shared memory, loaded CH rows at a time (one load latency per
// chunk), and the lanes share each elimination step's (row, column) updates.
//
// The reduced matrix is itself a structured matrix of the same family
// (SPEC.md: "block tridiagonal (no corner) or lower bidiagonal plus corner"):
// block tridiagonal with k x k blocks, or an ABD-style block row layout with a
// corner; it is assembled in the reference storage layout and solved by the
// same kernels recursively, ending in a one-warp bordered band solve
// (solve_sequential, src/seqref.cpp:12-93).
#pragma once

#include "psg_common.cuh"

namespace psg {

// Structured matrix view in the reference storage layout (structmat.hpp:16-31).
struct SMView {
  int kind, n, m, s, r;
  const double* data;
  const double* corner;
  int cr, cc;
};

__device__ __forceinline__ long sm_band_off(int n, int s, int d) {
  long off = 0;
  for (int b = -s; b < d; ++b) off += n - (b < 0 ? -b : b);
  return off;
}

// Closed form of abd_row_offset (src/structmat.cpp:47-54) for s <= m: row 0 is
// left-clipped (m + r wide), rows 1..nb-2 are m + s + r wide.
__device__ __forceinline__ long sm_abd_off(const SMView& A, long b) {
  return b == 0 ? 0 : (long)A.m * (A.m + A.r) + (b - 1) * (long)A.m * (A.m + A.r + A.s);
}

// A(i, j) with structural zeros (StructuredMatrix::at, src/structmat.cpp:112-145).
__device__ __forceinline__ double sm_at(const SMView& A, long i, long j) {
  if (i < 0 || j < 0 || i >= A.n || j >= A.n) return 0.0;
  const int m = A.m;
  if (A.kind == 0) {
    const long d = j - i;
    if (d < -A.s || d > A.r) return 0.0;
    return __ldg(A.data + sm_band_off(A.n, A.s, (int)d) + (i - (d < 0 ? -d : 0)));
  }
  if (A.kind == 4) {  // CirculantLike: band d = (j - i) mod n, wrapped (src/structmat.cpp:103-107, 137-142)
    long dd = j - i;
    if (dd < 0) dd += A.n;
    if (!(dd <= A.r || A.n - dd <= A.s)) return 0.0;
    const long d = dd <= A.r ? dd : dd - A.n;
    return __ldg(A.data + (d + A.s) * (long)A.n + i);
  }
  if (A.kind == 1) {
    const long bi = i / m, bj = j / m;
    if (bi - bj > 1 || bj - bi > 1) return 0.0;
    const long off = bi == 0 ? 0 : (3 * bi - 1) * (long)m * m;
    const long blk = bi > 0 ? bj - bi + 1 : bj - bi;
    return __ldg(A.data + off + blk * m * m + (i - bi * m) * m + (j - bj * m));
  }
  const long b = i / m;
  const long c0 = b * m - A.s > 0 ? b * m - A.s : 0;
  const long c1 = b * m + m + A.r < A.n ? b * m + m + A.r : A.n;
  if (j >= c0 && j < c1) return __ldg(A.data + sm_abd_off(A, b) + (i - b * m) * (c1 - c0) + (j - c0));
  if (A.kind == 3 && i < A.cr && j >= A.n - A.cc) return __ldg(A.corner + i * A.cc + (j - (A.n - A.cc)));
  return 0.0;
}

// Per-partition plan entry (host-built from plan_partition, src/partition.cpp:52-105).
struct GPart {
  int b, L;    // body rows [b, b+L)
  int ls, rs;  // left / right separator start row (-1: none)
};

struct GenArgs {
  SMView A;
  const GPart* part;
  int p, k;
  int es, er;          // scalar envelope of A (src/structmat.cpp:271-280)
  const double* f;     // rhs, indexed by global row (condense / backsolve)
  const double* xsep;  // separator values, k per separator, separator index order (backsolve)
  int has_corner;
  double* blocks;      // factor out: 4 k*k per partition (alpha1, alpha2, beta, gamma)
  double* kr;          // condense out: 2k per partition (top, bottom)
  double* x;           // backsolve out, indexed by global row
  double* scratch;     // backsolve: (er+2) doubles per body row
  DevStatus* status;   // zero-pivot attribution (level 0 only)
};

constexpr int kGenCH = 16;    // rows per staged chunk
constexpr int kGenMaxW = 32;  // band width es+1+er (Babd m=8 s=8 r=0: 23; its reduced system: 31)
constexpr int kGenMaxK = 8;   // separator size
constexpr int kGenMaxNR = 2 * kGenMaxK;

// Elimination state of one sweep in shared memory.
struct GenSweepSmem {
  double ring[kGenMaxW + kGenCH][kGenMaxW + kGenMaxNR];  // rows x: band (es+1+er) | rhs (nr)
  double tail[kGenMaxW][kGenMaxW + kGenMaxNR];           // last finished rows: U (d=0..er) | rhs
  double mu[32];
};

// Row x of the (possibly reversed) body: value at band offset d.
struct BodyMap {
  int b, L;
  bool rev;
  __device__ __forceinline__ long row(int x) const { return rev ? (long)b + L - 1 - x : (long)b + x; }
};

// One windowed no-pivot band LU sweep over the body (top-down on the mapped
// rows).  On return tail[] holds, for the last R rows of the mapped body, the
// solution rows of B^-1 X (columns 0..nr-1) in tail[x % kGenMaxW][w + c].
// MODE 2 instead streams each finished row (U d=0..er, g) to scratch.
// Returns false when a pivot vanished.
template <int MODE>
__device__ bool gen_sweep(const GenArgs& g, const GPart& P, const BodyMap& bm, int es, int er, int nr, int R,
                          const double* xl, const double* xr, GenSweepSmem& sm) {
  const int lane = threadIdx.x & 31;
  const int w = es + 1 + er;
  const int L = bm.L;
  const int W = es + 1 + kGenCH;  // ring rows
  int loaded = 0;
  bool ok = true;
  auto load_rows = [&](int upto) {
    const int x0 = loaded, x1 = min(L, upto);
    const int cols = w + nr;
    for (int idx = lane; idx < (x1 - x0) * cols; idx += 32) {
      const int dx = idx % (x1 - x0), col = idx / (x1 - x0);
      const int x = x0 + dx;
      const long gr = bm.row(x);
      double v;
      if (col < w) {
        const int d = col - es;  // mapped column x + d
        const int xc = x + d;
        v = (xc >= 0 && xc < L) ? sm_at(g.A, gr, bm.row(xc)) : 0.0;
      } else {
        const int c = col - w;
        if (MODE == 0) {
          v = c < g.k ? (P.ls >= 0 ? sm_at(g.A, gr, (long)P.ls + c) : 0.0)
                      : (P.rs >= 0 ? sm_at(g.A, gr, (long)P.rs + (c - g.k)) : 0.0);
        } else {
          v = __ldg(g.f + gr);
          if (MODE == 2) {
            for (int t = 0; t < g.k; ++t) {
              if (P.ls >= 0) v = fma(-sm_at(g.A, gr, (long)P.ls + t), xl[t], v);
              if (P.rs >= 0) v = fma(-sm_at(g.A, gr, (long)P.rs + t), xr[t], v);
            }
          }
        }
      }
      sm.ring[x % W][col] = v;
    }
    loaded = x1;
  };
  load_rows(min(L, es + 1 + kGenCH));
  __syncwarp();
  for (int k = 0; k < L; ++k) {
    if (loaded < L && k + es >= loaded) {
      load_rows(loaded + kGenCH);
      __syncwarp();
    }
    double* rk = sm.ring[k % W];
    const double piv = rk[es];
    if (piv == 0.0 || !isfinite(piv)) ok = false;
    const int ni = min(es, L - 1 - k);
    if (lane < ni) {
      double* ri = sm.ring[(k + 1 + lane) % W];
      const double mu = ri[es - 1 - lane] / piv;
      ri[es - 1 - lane] = 0.0;
      sm.mu[lane] = mu;
    }
    __syncwarp();
    const int nj = min(er, L - 1 - k) + nr;  // band columns k+1..k+er, then the rhs
    for (int idx = lane; idx < ni * nj; idx += 32) {
      const int i = idx / nj + 1, j = idx % nj;
      double* ri = sm.ring[(k + i) % W];
      const double mu = sm.mu[i - 1];
      if (j < min(er, L - 1 - k)) {
        ri[es - i + j + 1] = fma(-mu, rk[es + j + 1], ri[es - i + j + 1]);
      } else {
        const int c = j - min(er, L - 1 - k);
        ri[w + c] = fma(-mu, rk[w + c], ri[w + c]);
      }
    }
    // finished row k: keep it (tail ring) or stream it (backsolve scratch)
    if (MODE == 2) {
      double* sc = g.scratch + (long)(bm.b + k) * (er + 2);
      for (int d = lane; d <= er; d += 32) sc[d] = rk[es + d];
      if (lane == 0) sc[er + 1] = rk[w];
    } else if (k >= L - R) {
      double* tr = sm.tail[k % kGenMaxW];
      for (int d = lane; d <= er; d += 32) tr[d] = rk[es + d];
      for (int c = lane; c < nr; c += 32) tr[w + c] = rk[w + c];
    }
    __syncwarp();
  }
  if (MODE != 2) {
    // back-substitute the last R rows inside the tail (rows beyond L are zero)
    for (int x = L - 1; x >= L - R; --x) {
      double* tr = sm.tail[x % kGenMaxW];
      for (int c = lane; c < nr; c += 32) {
        double acc = tr[w + c];
        for (int d = 1; d <= er && x + d < L; ++d) acc = fma(-tr[d], sm.tail[(x + d) % kGenMaxW][w + c], acc);
        tr[w + c] = acc / tr[0];
      }
      __syncwarp();
    }
  }
  return ok;
}

// FACTOR (MODE 0) and CONDENSE (MODE 1): one warp per (partition, end).
// end 0 = top-down sweep -> last rows -> B1 terms (alpha2, beta | kr bottom),
// end 1 = bottom-up sweep -> first rows -> C0 terms (alpha1, gamma | kr top).
template <int MODE>
__global__ void __launch_bounds__(32) gen_ends_kernel(GenArgs g) {
  __shared__ GenSweepSmem sm;
  const int lane = threadIdx.x & 31;
  const long task = (long)blockIdx.x;
  if (task >= 2L * g.p) return;
  const int i = (int)(task >> 1), end = (int)(task & 1);
  const GPart P = g.part[i];
  const int k = g.k;
  const bool rev = end == 1;
  const int es = rev ? g.er : g.es, er = rev ? g.es : g.er;
  const int nr = MODE == 0 ? 2 * k : 1;
  const int R = min(P.L, kGenMaxW);  // rows whose solution the couplings can touch
  BodyMap bm{P.b, P.L, rev};
  const bool ok = gen_sweep<MODE>(g, P, bm, es, er, nr, R, nullptr, nullptr, sm);
  if (!ok && lane == 0 && g.status) status_pivot(g.status, i);
  // solution row of original body row xo (must be within the kept tail)
  auto sol = [&](int xo, int c) -> double {
    const int x = rev ? P.L - 1 - xo : xo;
    return sm.tail[x % kGenMaxW][(es + 1 + er) + c];
  };
  if (MODE == 0) {
    double* out = g.blocks + (long)i * 4 * k * k;  // alpha1 | alpha2 | beta | gamma
    const int sep = end == 0 ? P.rs : P.ls;
    for (int idx = lane; idx < 2 * k * k; idx += 32) {
      const int t = (idx / k) % k, u = idx % k, which = idx / (k * k);  // which: 0 -> B0 col block, 1 -> C1
      double acc = 0.0;
      if (sep >= 0) {
        for (int q = 0; q < R; ++q) {
          const int xo = end == 0 ? P.L - R + q : q;
          // B1[t][xo] (end 0) or C0[t][xo] (end 1): the separator row's entry in body column xo
          acc = fma(sm_at(g.A, (long)sep + t, (long)P.b + xo), sol(xo, which * k + u), acc);
        }
      }
      if (end == 0) {
        if (which == 1)
          out[1 * k * k + t * k + u] = (sep >= 0 ? sm_at(g.A, (long)sep + t, (long)sep + u) : 0.0) - acc;  // alpha2
        else
          out[2 * k * k + t * k + u] = -acc;  // beta
      } else {
        if (which == 0)
          out[0 * k * k + t * k + u] = -acc;  // alpha1
        else
          out[3 * k * k + t * k + u] = -acc;  // gamma
      }
    }
  } else {
    double* out = g.kr + (long)i * 2 * k;  // top | bottom
    const int sep = end == 0 ? P.rs : P.ls;
    for (int t = lane; t < k; t += 32) {
      double acc = 0.0;
      if (sep >= 0)
        for (int q = 0; q < R; ++q) {
          const int xo = end == 0 ? P.L - R + q : q;
          acc = fma(sm_at(g.A, (long)sep + t, (long)P.b + xo), sol(xo, 0), acc);
        }
      out[(end == 0 ? k : 0) + t] = -acc;
    }
  }
}

// BACKSOLVE: one warp per partition: forward sweep streaming U rows and the
// eliminated rhs to scratch, then back substitution; also writes the
// separator values owned by this partition (its right separator, and the
// first separator for corner plans).
__global__ void __launch_bounds__(32) gen_backsolve_kernel(GenArgs g) {
  __shared__ GenSweepSmem sm;
  __shared__ double xs[2 * kGenMaxK];
  const int lane = threadIdx.x;
  const int i = blockIdx.x;
  const GPart P = g.part[i];
  const int k = g.k;
  const int lsi = g.has_corner ? i : i - 1;  // separator indices
  const int rsi = g.has_corner ? i + 1 : i;
  if (lane < k) {
    xs[lane] = P.ls >= 0 ? g.xsep[(long)lsi * k + lane] : 0.0;
    xs[k + lane] = P.rs >= 0 ? g.xsep[(long)rsi * k + lane] : 0.0;
  }
  __syncwarp();
  BodyMap bm{P.b, P.L, false};
  const bool ok = gen_sweep<2>(g, P, bm, g.es, g.er, 1, 0, xs, xs + k, sm);
  if (!ok && lane == 0 && g.status) status_pivot(g.status, i);
  // back substitution: y_x = (g_x - sum_d U_x[d] y_{x+d}) / U_x[0], er-wide window in registers (lane 0)
  const int er = g.er;
  double win[kGenMaxW];
#pragma unroll
  for (int d = 0; d < kGenMaxW; ++d) win[d] = 0.0;
  bool finite = true;
  if (lane == 0) {
    for (int x = P.L - 1; x >= 0; --x) {
      const double* sc = g.scratch + (long)(P.b + x) * (er + 2);
      double acc = sc[er + 1];
      for (int d = 1; d <= er; ++d) acc = fma(-sc[d], win[d - 1], acc);
      const double y = acc / sc[0];
      finite &= isfinite(y);
      for (int d = kGenMaxW - 1; d > 0; --d) win[d] = win[d - 1];
      win[0] = y;
      g.x[(long)P.b + x] = y;
    }
    if (!finite && g.status) status_nonfinite(g.status, i);
  }
  if (lane < k) {
    if (P.rs >= 0) g.x[(long)P.rs + lane] = xs[k + lane];
    if (g.has_corner && i == 0 && P.ls >= 0) g.x[(long)P.ls + lane] = xs[lane];
  }
}

// ---------------------------------------------------------------------------
// Reduced system assembly in a structured layout (the parfact.cpp:72-127
// scatter, written as the next level's StructuredMatrix data).
//   no corner: BlockTridiagonal, m = k, N = p-1 block rows
//   corner   : ABD row layout m = k, s = k, r = k (block tridiagonal) + k x k
//              corner, N = p+1 block rows
// ---------------------------------------------------------------------------
__global__ void gen_assemble_T_kernel(GenArgs g, double* __restrict__ T, double* __restrict__ Tcorner) {
  const int k = g.k, kk = k * k;
  const int q = g.has_corner ? g.p + 1 : g.p - 1;
  const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;  // one thread per (block row, entry)
  if (e >= (long)q * kk) return;
  const int j = (int)(e / kk), t = (int)(e % kk) / k, u = (int)(e % kk) % k;
  const double* B = g.blocks;
  auto blk = [&](int part, int which) { return B[(long)part * 4 * kk + which * kk + t * k + u]; };
  double sub = 0.0, dia = 0.0, sup = 0.0;
  if (!g.has_corner) {
    // separator j between partitions j (right sep) and j+1 (left sep)
    sub = blk(j, 2);                      // beta^(j)
    dia = blk(j, 1) + blk(j + 1, 0);      // alpha2^(j) + alpha1^(j+1)
    sup = blk(j + 1, 3);                  // gamma^(j+1)
    // BlockTridiagonal layout: row j at (3j-1)k^2 (j > 0): [sub | diag | super]
    const long off = j == 0 ? 0 : (3L * j - 1) * kk;
    const int dblk = j > 0 ? 1 : 0;
    if (j > 0) T[off + t * k + u] = sub;
    T[off + (long)dblk * kk + t * k + u] = dia;
    if (j < q - 1) T[off + (long)(dblk + 1) * kk + t * k + u] = sup;
  } else {
    // separator j: right sep of partition j-1, left sep of partition j
    if (j >= 1) {
      sub = blk(j - 1, 2);  // beta^(j-1)
      dia += blk(j - 1, 1);  // alpha2^(j-1)
    }
    if (j <= g.p - 1) {
      dia += blk(j, 0);  // alpha1^(j)
      sup = blk(j, 3);   // gamma^(j)
    }
    if (j == 0) {  // the first separator's own diagonal block and the corner (parfact.cpp:94-104)
      const GPart P0 = g.part[0];
      dia += sm_at(g.A, (long)P0.ls + t, (long)P0.ls + u);
      const GPart PL = g.part[g.p - 1];
      Tcorner[t * k + u] = sm_at(g.A, (long)P0.ls + t, (long)PL.rs + u);
    }
    // ABD layout with m = s = r = k: row 0 spans blocks [0, 2), rows 1..q-2 [j-1, j+2), row q-1 [q-2, q)
    const long off = j == 0 ? 0 : (long)k * 2 * k + (long)(j - 1) * k * 3 * k;
    const int width = (j == 0 || j == q - 1) ? 2 * k : 3 * k;
    double* row = T + off + (long)t * width;
    if (j == 0) {
      row[u] = dia;
      row[k + u] = sup;
    } else {
      row[u] = sub;
      row[k + u] = dia;
      if (j < q - 1) row[2 * k + u] = sup;
    }
  }
}

// next-level rhs: f at the separator rows plus the kept contributions
__global__ void gen_assemble_rhs_kernel(GenArgs g, const int* __restrict__ sep_start, double* __restrict__ rhs) {
  const int k = g.k;
  const int q = g.has_corner ? g.p + 1 : g.p - 1;
  const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e >= (long)q * k) return;
  const int j = (int)(e / k), t = (int)(e % k);
  double v = __ldg(g.f + (long)sep_start[j] + t);
  // reference order: original entry, then partitions in index order (parfact.cpp:205-214)
  if (!g.has_corner) {
    v += g.kr[(long)j * 2 * k + k + t];        // partition j, right separator (bottom)
    v += g.kr[(long)(j + 1) * 2 * k + t];      // partition j+1, left separator (top)
  } else {
    if (j >= 1) v += g.kr[(long)(j - 1) * 2 * k + k + t];
    if (j <= g.p - 1) v += g.kr[(long)j * 2 * k + t];
  }
  rhs[e] = v;
}

// ---------------------------------------------------------------------------
// Direct solve of a small structured system by one warp: the reference's
// bordered band elimination (solve_sequential, src/seqref.cpp:12-93): band LU
// over the first nb = n - K rows with K spike columns, condensed K x K tail,
// partial-pivot dense LU of the tail, back substitution.  Scratch: band
// nb x w, spike nb x K, tail K x K + K.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32) gen_direct_kernel(SMView A, int es, int er, int K, const double* __restrict__ f,
                                                        double* __restrict__ x, double* __restrict__ work,
                                                        DevStatus* st) {
  const int lane = threadIdx.x;
  const int n = A.n, nb = n - K, w = es + 1 + er;
  double* band = work;                        // nb x w
  double* spike = band + (long)nb * w;        // nb x K
  double* rhs = spike + (long)nb * K;         // n
  double* tail = rhs + n;                     // K x K
  double* trhs = tail + (long)K * K;          // K
  double* row = trhs + K;                     // n (tail row scratch)
  for (long idx = lane; idx < (long)nb * w; idx += 32) {
    const long i = idx / w, jj = idx % w - es;
    const long j = i + jj;
    band[idx] = (j >= 0 && j < nb) ? sm_at(A, i, j) : 0.0;
  }
  for (long idx = lane; idx < (long)nb * K; idx += 32) spike[idx] = sm_at(A, idx / K, nb + idx % K);
  for (long i = lane; i < n; i += 32) rhs[i] = f[i];
  __syncwarp();
  bool ok = true;
  for (int k = 0; k < nb; ++k) {
    const double d = band[(long)k * w + es];
    if (d == 0.0) ok = false;
    const int ilim = min(nb - 1, k + es);
    for (int i = k + 1; i <= ilim; ++i) {
      const double e = band[(long)i * w + (k - i + es)];
      if (e == 0.0) continue;
      const double mu = e / d;
      const int jlim = min(nb - 1, k + er);
      for (int j = k + 1 + lane; j <= jlim; j += 32)
        band[(long)i * w + (j - i + es)] -= mu * band[(long)k * w + (j - k + es)];
      for (int q = lane; q < K; q += 32) spike[(long)i * K + q] -= mu * spike[(long)k * K + q];
      if (lane == 0) rhs[i] -= mu * rhs[k];
      __syncwarp();
    }
  }
  for (int t = 0; t < K; ++t) {
    const int i = nb + t;
    for (int j = lane; j < n; j += 32) row[j] = sm_at(A, i, j);
    __syncwarp();
    double rv = f[i];
    for (int k = (i - es - K > 0 ? i - es - K : 0); k < nb; ++k) {
      const double e = row[k];
      if (e == 0.0) continue;
      const double mu = e / band[(long)k * w + es];
      __syncwarp();
      if (lane == 0) row[k] = 0.0;
      const int jlim = min(nb - 1, k + er);
      for (int j = k + 1 + lane; j <= jlim; j += 32) row[j] -= mu * band[(long)k * w + (j - k + es)];
      for (int q = lane; q < K; q += 32) row[nb + q] -= mu * spike[(long)k * K + q];
      rv -= mu * rhs[k];
      __syncwarp();
    }
    for (int q = lane; q < K; q += 32) tail[(long)t * K + q] = row[nb + q];
    if (lane == 0) trhs[t] = rv;
    __syncwarp();
  }
  // dense LU with partial pivoting of the K x K tail (src/dense.cpp:78-120), lane 0
  if (lane == 0 && K > 0) {
    for (int k = 0; k < K; ++k) {
      int piv = k;
      double best = fabs(tail[k * K + k]);
      for (int i = k + 1; i < K; ++i)
        if (fabs(tail[i * K + k]) > best) {
          best = fabs(tail[i * K + k]);
          piv = i;
        }
      if (best == 0.0) ok = false;
      if (piv != k) {
        for (int j = 0; j < K; ++j) {
          const double tmp = tail[k * K + j];
          tail[k * K + j] = tail[piv * K + j];
          tail[piv * K + j] = tmp;
        }
        const double tr = trhs[k];
        trhs[k] = trhs[piv];
        trhs[piv] = tr;
      }
      for (int i = k + 1; i < K; ++i) {
        const double m = tail[i * K + k] / tail[k * K + k];
        for (int j = k + 1; j < K; ++j) tail[i * K + j] -= m * tail[k * K + j];
        trhs[i] -= m * trhs[k];
      }
    }
    for (int i = K - 1; i >= 0; --i) {
      double acc = trhs[i];
      for (int j = i + 1; j < K; ++j) acc -= tail[i * K + j] * trhs[j];
      trhs[i] = acc / tail[i * K + i];
      x[nb + i] = trhs[i];
    }
  }
  __syncwarp();
  if (lane == 0) {
    for (int k = nb - 1; k >= 0; --k) {
      double acc = rhs[k];
      for (int j = k + 1; j <= min(nb - 1, k + er); ++j) acc -= band[(long)k * w + (j - k + es)] * x[j];
      for (int q = 0; q < K; ++q) acc -= spike[(long)k * K + q] * x[nb + q];
      x[k] = acc / band[(long)k * w + es];
    }
  }
  if (!ok && lane == 0 && st) status_nonfinite(st, 0);
}

}  // namespace psg
