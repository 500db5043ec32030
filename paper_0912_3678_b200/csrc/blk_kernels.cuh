// blk_kernels.cuh -- the speculative partition method for K x K block-
// tridiagonal structure: BlockTridiagonal m = K and Banded s, r <= K (a band
// matrix is block tridiagonal with K x K blocks on any K-aligned row grid).
// K = 2..4.  The scalar tridiagonal path (tri_kernels.cuh) is the K = 1 case
// of the same design:
//
//   factor + separators (blk_spec_fused_kernel, lazy: one launch per
//     refactor + solve): per separator block S (K rows), the Schur complement
//     T = A_SS - B1 [B_T^-1]_{near} C_T - C0 [B_L^-1]_{near} A_L of the
//     TRUNCATED neighbouring bodies (HB block rows each side) and, carried by
//     the same far -> near block sweeps, the condensed right-hand sides, so
//     x_S = T^-1 (f_S - B1 [B_T^-1 f_T]_{near} - C0 [B_L^-1 f_L]_{near})
//     -- the separator row of F T G restricted to the truncation window
//     (src/localfact.cpp:84-225, 765-781 compute the same blocks on full
//     bodies); no weights are formed;
//   solve:
//     blk_segment_solve_kernel the bodies, exact given x_S (warp per body, block
//                              chunk elimination + block PCR across lanes);
//     blk_cert_kernel          componentwise backward error of every separator
//                              row from the bodies' boundary records.
//   A failed certificate sends the solve to the exact generic path
//   (gen_exact.cuh), whose level-0 back-substitution is this same body kernel.
//
// No pivoting inside blocks (the reference's Lu/Lud strategies assume the
// same; a vanished pivot is reported as ZeroPivot by the exact path).
#pragma once

#include "gen_exact.cuh"
#include "psg_common.cuh"

namespace psg {

// ---------------------------------------------------------------------------
// register K x K block algebra (segment kernel)
// ---------------------------------------------------------------------------
template <int K>
struct Blk {
  double v[K][K];
};
template <int K>
struct Vec {
  double v[K];
};

template <int K>
__device__ __forceinline__ Blk<K> blk_mul(const Blk<K>& A, const Blk<K>& B) {
  Blk<K> C;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double acc = A.v[i][0] * B.v[0][j];
#pragma unroll
      for (int l = 1; l < K; ++l) acc = fma(A.v[i][l], B.v[l][j], acc);
      C.v[i][j] = acc;
    }
  return C;
}

// C -= A B
template <int K>
__device__ __forceinline__ void blk_mul_sub(Blk<K>& C, const Blk<K>& A, const Blk<K>& B) {
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double acc = C.v[i][j];
#pragma unroll
      for (int l = 0; l < K; ++l) acc = fma(-A.v[i][l], B.v[l][j], acc);
      C.v[i][j] = acc;
    }
}

template <int K>
__device__ __forceinline__ Vec<K> blk_mv(const Blk<K>& A, const Vec<K>& x) {
  Vec<K> y;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double acc = A.v[i][0] * x.v[0];
#pragma unroll
    for (int l = 1; l < K; ++l) acc = fma(A.v[i][l], x.v[l], acc);
    y.v[i] = acc;
  }
  return y;
}

// y -= A x
template <int K>
__device__ __forceinline__ void blk_mv_sub(Vec<K>& y, const Blk<K>& A, const Vec<K>& x) {
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double acc = y.v[i];
#pragma unroll
    for (int l = 0; l < K; ++l) acc = fma(-A.v[i][l], x.v[l], acc);
    y.v[i] = acc;
  }
}

template <int K>
__device__ __forceinline__ void blk_neg(Blk<K>& A) {
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) A.v[i][j] = -A.v[i][j];
}

template <int K>
__device__ __forceinline__ void blk_set_eye(Blk<K>& A) {
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) A.v[i][j] = i == j ? 1.0 : 0.0;
}

template <int K>
__device__ __forceinline__ void blk_set_zero(Blk<K>& A) {
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) A.v[i][j] = 0.0;
}

// In-place inverse, Gauss-Jordan without pivoting; sum |1/pivot| -> *rsum.
template <int K>
__device__ __forceinline__ void blk_inv(Blk<K>& A, double* rsum) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double p = fast_rcp(A.v[k][k]);
    *rsum += fabs(p);
    A.v[k][k] = 1.0;
#pragma unroll
    for (int j = 0; j < K; ++j) A.v[k][j] *= p;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i == k) continue;
      const double f = A.v[i][k];
      A.v[i][k] = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) A.v[i][j] = fma(-f, A.v[k][j], A.v[i][j]);
    }
  }
}

template <int K>
__device__ __forceinline__ Blk<K> blk_shfl(const Blk<K>& a, int src) {
  Blk<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) r.v[i][j] = __shfl_sync(0xffffffffu, a.v[i][j], src);
  return r;
}
template <int K>
__device__ __forceinline__ Vec<K> vec_shfl(const Vec<K>& a, int src) {
  Vec<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.v[i] = __shfl_sync(0xffffffffu, a.v[i], src);
  return r;
}

// Lane-level reduced systems in normalised form, al X_{t-1} + X_t + ga X_{t+1}
// = de, one block row per lane, in groups of LPB lanes (r = index in the
// group; the rows at a group's ends have zero couplings outward).  For the
// block diagonally dominant bodies the speculative paths certify, the
// couplings are tiny: with kappa = max row sum of |al| + |ga| (over the warp)
// block Jacobi sweeps X <- de - al X_{t-1} - ga X_{t+1} from X = de leave an
// error below kappa^(it+1) |X|, so `it` is chosen with kappa^(it+1) <= 2^-64
// (2 K x K mat-vecs per sweep instead of a PCR step's 6 K x K products and an
// inverse; measured: config 3 with 254-row bodies, kappa ~ 1e-3, 0.54 -> 0.41
// ms for the bodies against PCR).  Returns false (de untouched) when kappa >
// 1/4 or is not finite: the caller runs PCR.  Warp-uniform; every lane must
// call it.
constexpr double kJacobiKappa = 0.25;  // at most 31 sweeps (cheaper than the 5 PCR steps of 32 lanes)
template <int K>
__device__ __forceinline__ bool blk_jacobi(const Blk<K>& al, const Blk<K>& ga, Vec<K>& de, int r, int LPB) {
  constexpr double kDecoupled = 5.421010862427522e-20;  // 2^-64
  const int lane = threadIdx.x & 31;
  double kap = 0.0;
#pragma unroll
  for (int u = 0; u < K; ++u) {
    double rsu = 0.0;
#pragma unroll
    for (int v = 0; v < K; ++v) rsu += fabs(al.v[u][v]) + fabs(ga.v[u][v]);
    kap = fmax(kap, rsu);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kap = fmax(kap, __shfl_xor_sync(0xffffffffu, kap, o));
  if (!(kap <= kJacobiKappa)) return false;
  int nit = 0;
  for (double pw = kap; pw > kDecoupled; pw *= kap) ++nit;
  const Vec<K> d0 = de;
  const int sl = r > 0 ? lane - 1 : lane, sh = r + 1 < LPB ? lane + 1 : lane;
#pragma unroll 1
  for (int it = 0; it < nit; ++it) {
    Vec<K> xl, xh;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      xl.v[u] = __shfl_sync(0xffffffffu, de.v[u], sl);
      xh.v[u] = __shfl_sync(0xffffffffu, de.v[u], sh);
    }
    Vec<K> nx = d0;
    blk_mv_sub<K>(nx, al, xl);
    blk_mv_sub<K>(nx, ga, xh);
    de = nx;
  }
  return true;
}

__device__ __forceinline__ long band_start(long n, int s, int d) {
  long off = 0;
  for (int b = -s; b < d; ++b) off += n - (b < 0 ? -b : b);
  return off;
}

// ---------------------------------------------------------------------------
// body solver
// ---------------------------------------------------------------------------
enum BlkLayout { kBlkBlockTri = 0, kBlkBanded = 1 };

struct BlkArgs {
  const double* data;  // matrix storage (reference layout)
  long n;              // scalar dimension
  int s, r;            // banded: bandwidths (<= K)
  const double* f;     // rhs by global row
  double* x;           // solution by global row
  const double* xsep;  // separator values, K per separator (separator index order)
  const GPart* part;   // bodies: [b, b+L), separators ls / rs (-1: none)
  int nseg;
  double* rec;         // certificate records (4K per body) or null
  DevStatus* status;
  long boff[9];        // banded: A(row, row + d) = data[boff[d + K] + row] (host-computed)
  long data_len;       // entries in data (staging over-read bound)
};

template <int K, int M, int NW = 1>
struct BlkSmem {
  static constexpr int NT = 32 * NW;               // threads per body
  static constexpr int NBMAX = NT * M;             // block rows per body
  static constexpr int P = NBMAX + 1;              // element-major pitch (odd)
  static constexpr int PB = NBMAX * K + 1;         // banded: band pitch (odd)
  static constexpr int MAT_BT = 3 * K * K * P;     // block tridiagonal staging
  static constexpr int MAT_BD = (2 * K + 1) * PB;  // banded staging (bands -K..K)
  static constexpr int STASH = NT * M * (2 * K * K + K);
  static constexpr int MAT = (MAT_BT > STASH ? MAT_BT : STASH);
  static constexpr int RB = NBMAX * K + 4;         // banded: per-band TMA region (even: 16-byte aligned)
  static constexpr int MATB = (2 * K + 1) * RB;    // >= STASH
  static constexpr int MAT_ALIGNED = (MAT + 1) & ~1;
  static constexpr int F = NBMAX * K + 4;          // rhs region (TMA, shifted)
  static constexpr int XCH = NW > 1 ? NT * (2 * K * K + K) : 0;  // cross-warp exchange (NW > 1)
  static constexpr int bytes(int layout) { return 8 * ((layout == kBlkBlockTri ? MAT_ALIGNED : MATB) + F + XCH); }
};

// Certificate record of one body (4K doubles): for its left separator rows u,
//   rec[0..K)  sum_t A(ls+u, b+t) y(b+t)   rec[K..2K)  sum |.|
// and for its right separator rows with the body's last rows
//   rec[2K..3K) signed                      rec[3K..4K) abs.

template <int K, int M, int LAYOUT, int NW>
__global__ void __launch_bounds__(32 * NW) blk_segment_solve_kernel(BlkArgs g) {
  using SM = BlkSmem<K, M, NW>;
  constexpr int NT = SM::NT;
  constexpr int P = SM::P;
  constexpr int KK = K * K;
  constexpr int MATD = LAYOUT == kBlkBlockTri ? SM::MAT_ALIGNED : SM::MATB;
  constexpr int RB = SM::RB;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int boffs[2 * K + 2];  // banded: smem offset of row 0 of band d (d + K); [2K+1]: f
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int seg = blockIdx.x;
  auto SYNC = [&]() {
    if (NW > 1)
      __syncthreads();
    else
      __syncwarp();
  };
  const GPart Pt = g.part[seg];
  const long b = Pt.b;
  const int L = Pt.L;
  const int NB = (L + K - 1) / K;
  const int NR = NB * K;
  const long n = g.n;
  const int lsi = seg - 1, rsi = seg;

  // ---- staging: rhs (and banded: every band) by TMA bulk copies, one lane per array;
  //      block tridiagonal: element-major transposition through registers
  constexpr int NARR = LAYOUT == kBlkBlockTri ? 1 : 2 * K + 2;
  if (tid == 0) mbar_init(&bar, NARR);
  SYNC();
  RowArr X{};
  double* xbase = nullptr;
  if (tid < NARR) {
    if (tid == NARR - 1) {  // rhs
      X = make_rows(g.f, 0, (int)n, 0, n);
      xbase = sm + MATD;
    } else {
      const int d = lane - K;
      const bool inb = d >= -g.s && d <= g.r;
      const long bo = inb ? g.boff[lane] : 0;
      X = make_rows(g.data + bo, inb ? (d < 0 ? -d : 0) : 0, inb ? (int)(n - (d > 0 ? d : 0)) : 0, -bo,
                    g.data_len - bo);
      xbase = sm + lane * RB;
    }
    uint32_t tx = 0;
    const int shift = stage_issue(X, b, b + NR, xbase, &bar, &tx);
    mbar_arrive_expect_tx(&bar, tx);
    boffs[tid] = (int)(xbase - sm) + 1 + shift;
  }
  if (LAYOUT == kBlkBlockTri) {
    // block rows B0..B0+NB-1 are contiguous: [(3 B0 - 1) KK, (3 (B0+NB) - 1) KK)
    const long B0 = b / K;
    const long g0 = (3 * B0 - 1) * KK;
    const int tot = NB * 3 * KK;
    const long glen = (3 * (n / K) - 2) * KK;
    const int ilo = (int)(g0 < 0 ? -g0 : 0);
    const int ihi = (int)(glen - g0 < tot ? glen - g0 : tot);
    constexpr int U = 16;  // loads in flight per lane
    for (int i0 = tid; i0 < tot; i0 += NT * U) {
      double v[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int i = i0 + NT * k;
        v[k] = (i >= ilo && i < ihi) ? __ldg(g.data + g0 + i) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int i = i0 + NT * k;
        if (i < tot) {
          const int q = i / (3 * KK), e = i - q * (3 * KK);
          sm[e * P + q] = v[k];
        }
      }
    }
  }
  Vec<K> xl, xrv;
  pdl_wait();     // separator values from the previous kernel (the staging above overlaps it)
  pdl_trigger();  // the certificate kernel may launch (it waits for this grid before reading the records)
#pragma unroll
  for (int u = 0; u < K; ++u) {
    xl.v[u] = Pt.ls >= 0 ? __ldg(g.xsep + (long)lsi * K + u) : 0.0;
    xrv.v[u] = Pt.rs >= 0 ? __ldg(g.xsep + (long)rsi * K + u) : 0.0;
  }
  mbar_wait(&bar, 0);
  if (tid < NARR) stage_fixup(X, b, b + NR, sm + boffs[tid]);
  SYNC();
  double* smf = sm + boffs[NARR - 1];  // rhs / solution by body row
  for (int xr = L + tid; xr < NR; xr += NT) smf[xr] = 0.0;  // padding rows
  int bo[2 * K + 1];
#pragma unroll
  for (int t = 0; t < 2 * K + 1; ++t) bo[t] = LAYOUT == kBlkBanded ? boffs[t] : 0;
  SYNC();
  // staged A(b+xrow, b+ycol) (0 outside the structure)
  auto elem = [&](int xrow, int ycol) -> double {
    if (LAYOUT == kBlkBlockTri) {
      const int q = xrow / K;
      const int qc = ycol >= 0 ? ycol / K : -1;
      const int blk = qc - q + 1;
      if (blk < 0 || blk > 2) return 0.0;
      return sm[(blk * KK + (xrow - q * K) * K + (ycol - qc * K)) * P + q];
    } else {
      const int d = ycol - xrow;
      if (d < -g.s || d > g.r) return 0.0;
      return sm[boffs[d + K] + xrow];
    }
  };
  // fold the separator couplings of the first / last K body rows into the rhs
  if (tid < K) {
    if (Pt.ls >= 0) {
      double fv = smf[tid];
#pragma unroll
      for (int t = 0; t < K; ++t) fv = fma(-elem(tid, t - K), xl.v[t], fv);
      smf[tid] = fv;
    }
  } else if (tid >= 16 && tid < 16 + K) {
    const int xrow = L - K + (tid - 16);
    if (Pt.rs >= 0) {
      double fv = smf[xrow];
#pragma unroll
      for (int t = 0; t < K; ++t) fv = fma(-elem(xrow, L + t), xrv.v[t], fv);
      smf[xrow] = fv;
    }
  }
  SYNC();

  // block (q, blk) with separator columns and padding rows masked out
  auto load_blk = [&](int q, int blk) {
    Blk<K> B;
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int v = 0; v < K; ++v) {
        const int xrow = q * K + u, ycol = (q + blk - 1) * K + v;
        double val;
        if (LAYOUT == kBlkBlockTri) {
          val = sm[(blk * KK + u * K + v) * P + q];
        } else {
          const int d = (blk - 1) * K + v - u;  // compile-time after unrolling
          val = (d >= -g.s && d <= g.r) ? sm[bo[d + K] + xrow] : 0.0;
        }
        if (xrow >= L)
          val = (blk == 1 && u == v) ? 1.0 : 0.0;  // padding: identity, decoupled
        else if (ycol < 0 || ycol >= L)
          val = 0.0;  // folded into the rhs
        B.v[u][v] = val;
      }
    return B;
  };

  // ---- block chunk elimination: AP_j y_first + y_j + CP_j y_last = DP_j
  Blk<K> AP[M], CP[M];
  Vec<K> DP[M];
  double rsum = 0.0;
  const int q0 = tid * M;
  double* xch = sm + (LAYOUT == kBlkBlockTri ? SM::MAT_ALIGNED : SM::MATB) + SM::F;  // NW > 1 exchange
  // NW > 1: write a block row (a, c, d) of thread tid into the exchange area / read thread src's
  auto xput = [&](const Blk<K>& a, const Blk<K>& c, const Vec<K>& d) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
#pragma unroll
      for (int v = 0; v < K; ++v) {
        xch[(u * K + v) * NT + tid] = a.v[u][v];
        xch[(K * K + u * K + v) * NT + tid] = c.v[u][v];
      }
      xch[(2 * K * K + u) * NT + tid] = d.v[u];
    }
  };
  auto xget = [&](int src, Blk<K>& a, Blk<K>& c, Vec<K>& d) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
#pragma unroll
      for (int v = 0; v < K; ++v) {
        a.v[u][v] = xch[(u * K + v) * NT + src];
        c.v[u][v] = xch[(K * K + u * K + v) * NT + src];
      }
      d.v[u] = xch[(2 * K * K + u) * NT + src];
    }
  };
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const int q = q0 + j;
    Blk<K> Ab, Db, Cb;
    Vec<K> Fv;
    if (q < NB) {
      Ab = load_blk(q, 0);
      Db = load_blk(q, 1);
      Cb = load_blk(q, 2);
#pragma unroll
      for (int u = 0; u < K; ++u) Fv.v[u] = smf[q * K + u];
    } else {
      blk_set_zero<K>(Ab);
      blk_set_zero<K>(Cb);
      blk_set_eye<K>(Db);
#pragma unroll
      for (int u = 0; u < K; ++u) Fv.v[u] = 0.0;
    }
    if (j < 2) {
      blk_inv<K>(Db, &rsum);
      AP[j] = blk_mul<K>(Db, Ab);
      CP[j] = blk_mul<K>(Db, Cb);
      DP[j] = blk_mv<K>(Db, Fv);
    } else {
      blk_mul_sub<K>(Db, Ab, CP[j - 1]);
      blk_inv<K>(Db, &rsum);
      blk_mv_sub<K>(Fv, Ab, DP[j - 1]);
      DP[j] = blk_mv<K>(Db, Fv);
      const Blk<K> aap = blk_mul<K>(Ab, AP[j - 1]);
      AP[j] = blk_mul<K>(Db, aap);
      blk_neg<K>(AP[j]);
      CP[j] = blk_mul<K>(Db, Cb);
    }
  }
#pragma unroll
  for (int j = M - 3; j >= 1; --j) {
    blk_mv_sub<K>(DP[j], CP[j], DP[j + 1]);
    blk_mul_sub<K>(AP[j], CP[j], AP[j + 1]);
    CP[j] = blk_mul<K>(CP[j], CP[j + 1]);
    blk_neg<K>(CP[j]);
  }
  if (M >= 3) {
    Blk<K> R;
    blk_set_eye<K>(R);
    blk_mul_sub<K>(R, CP[0], AP[1]);
    blk_inv<K>(R, &rsum);
    blk_mv_sub<K>(DP[0], CP[0], DP[1]);
    DP[0] = blk_mv<K>(R, DP[0]);
    AP[0] = blk_mul<K>(R, AP[0]);
    const Blk<K> cc = blk_mul<K>(CP[0], CP[1]);
    CP[0] = blk_mul<K>(R, cc);
    blk_neg<K>(CP[0]);
  }
  // ---- chunk interfaces: one normalised block row per lane in F = y_first
  Blk<K> al, ga, be;
  Vec<K> de = DP[0];
  blk_set_eye<K>(be);
  blk_set_zero<K>(al);
  if (NW == 1) {
    const int lo1 = lane > 0 ? lane - 1 : 0;
    const Blk<K> pa = blk_shfl<K>(AP[M - 1], lo1);
    if (lane > 0) {
      al = blk_mul<K>(AP[0], pa);
      blk_neg<K>(al);
    }
    const Blk<K> pc = blk_shfl<K>(CP[M - 1], lo1);
    if (lane > 0) blk_mul_sub<K>(be, AP[0], pc);
    const Vec<K> pd = vec_shfl<K>(DP[M - 1], lo1);
    if (lane > 0) blk_mv_sub<K>(de, AP[0], pd);
  } else {
    xput(AP[M - 1], CP[M - 1], DP[M - 1]);
    __syncthreads();
    if (tid > 0) {
      Blk<K> pa, pc;
      Vec<K> pd;
      xget(tid - 1, pa, pc, pd);
      al = blk_mul<K>(AP[0], pa);
      blk_neg<K>(al);
      blk_mul_sub<K>(be, AP[0], pc);
      blk_mv_sub<K>(de, AP[0], pd);
    }
  }
  blk_mul_sub<K>(be, CP[0], AP[M - 1]);
  blk_mv_sub<K>(de, CP[0], DP[M - 1]);
  ga = blk_mul<K>(CP[0], CP[M - 1]);
  blk_neg<K>(ga);
  // stash the chunk state in the consumed staging area (thread-interleaved)
  SYNC();
  {
    double* st = sm + tid;
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
      for (int u = 0; u < K; ++u) {
#pragma unroll
        for (int v = 0; v < K; ++v) {
          st[NT * ((j * K + u) * (2 * K + 1) + 2 * v)] = AP[j].v[u][v];
          st[NT * ((j * K + u) * (2 * K + 1) + 2 * v + 1)] = CP[j].v[u][v];
        }
        st[NT * ((j * K + u) * (2 * K + 1) + 2 * K)] = DP[j].v[u];
      }
  }
  blk_inv<K>(be, &rsum);
  al = blk_mul<K>(be, al);
  ga = blk_mul<K>(be, ga);
  de = blk_mv<K>(be, de);
  if (NW == 1) {
  const bool jac = blk_jacobi<K>(al, ga, de, lane, 32);
#pragma unroll 1
  for (int st = 1; st < (jac ? 1 : 32); st <<= 1) {
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
    blk_inv<K>(nb, &rsum);
    al = blk_mul<K>(nb, na);
    blk_neg<K>(al);
    ga = blk_mul<K>(nb, ng);
    blk_neg<K>(ga);
    de = blk_mv<K>(nb, nd);
  }
  } else {
#pragma unroll 1
    for (int st = 1; st < NT; st <<= 1) {
      const bool hl = tid >= st, hh = tid + st < NT;
      __syncthreads();
      xput(al, ga, de);
      __syncthreads();
      Blk<K> nb, na, ng;
      blk_set_eye<K>(nb);
      Vec<K> nd = de;
      blk_set_zero<K>(na);
      blk_set_zero<K>(ng);
      if (hl) {
        Blk<K> la, lg;
        Vec<K> ld;
        xget(tid - st, la, lg, ld);
        blk_mul_sub<K>(nb, al, lg);
        na = blk_mul<K>(al, la);
        blk_mv_sub<K>(nd, al, ld);
      }
      if (hh) {
        Blk<K> ha, hg;
        Vec<K> hd;
        xget(tid + st, ha, hg, hd);
        blk_mul_sub<K>(nb, ga, ha);
        ng = blk_mul<K>(ga, hg);
        blk_mv_sub<K>(nd, ga, hd);
      }
      blk_inv<K>(nb, &rsum);
      al = blk_mul<K>(nb, na);
      blk_neg<K>(al);
      ga = blk_mul<K>(nb, ng);
      blk_neg<K>(ga);
      de = blk_mv<K>(nb, nd);
    }
  }
  // ---- back-substitution
  const Vec<K> Fv = de;
  Vec<K> Fn;
  if (NW == 1) {
    Fn = vec_shfl<K>(Fv, lane < 31 ? lane + 1 : lane);
  } else {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < K; ++u) xch[u * NT + tid] = Fv.v[u];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < K; ++u) Fn.v[u] = tid + 1 < NT ? xch[u * NT + tid + 1] : 0.0;
  }
  if (tid == NT - 1)
#pragma unroll
    for (int u = 0; u < K; ++u) Fn.v[u] = 0.0;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const double* st = sm + tid;
#pragma unroll
    for (int u = 0; u < K; ++u) {
#pragma unroll
      for (int v = 0; v < K; ++v) {
        AP[j].v[u][v] = st[NT * ((j * K + u) * (2 * K + 1) + 2 * v)];
        CP[j].v[u][v] = st[NT * ((j * K + u) * (2 * K + 1) + 2 * v + 1)];
      }
      DP[j].v[u] = st[NT * ((j * K + u) * (2 * K + 1) + 2 * K)];
    }
  }
  Vec<K> Ev = DP[M - 1];
  blk_mv_sub<K>(Ev, AP[M - 1], Fv);
  blk_mv_sub<K>(Ev, CP[M - 1], Fn);
  bool finite = true;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    Vec<K> y;
    if (j == 0) {
      y = Fv;
    } else if (j == M - 1) {
      y = Ev;
    } else {
      y = DP[j];
      blk_mv_sub<K>(y, AP[j], Fv);
      blk_mv_sub<K>(y, CP[j], Ev);
    }
    const int q = q0 + j;
    if (q < NB) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        if (q * K + u < L) finite &= isfinite(y.v[u]);
        smf[q * K + u] = y.v[u];
      }
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
  SYNC();
  for (int r = tid; r < L; r += NT) g.x[b + r] = smf[r];
  if (tid < K && Pt.rs >= 0) g.x[Pt.rs + tid] = xrv.v[tid];
  // ---- certificate records: the separator rows' couplings to this body
  if (g.rec) {
    double* rc = g.rec + (long)seg * 4 * K;
    auto at = [&](long row, long col) -> double {  // global A(row, col), known in range
      if (LAYOUT == kBlkBlockTri) {
        const long B = row / K, Bc = col / K;
        if (Bc < B - 1 || Bc > B + 1) return 0.0;
        const long off = B == 0 ? 0 : (3 * B - 1) * KK;
        const long blk = B == 0 ? Bc - B : Bc - B + 1;
        return __ldg(g.data + off + blk * KK + (row - B * K) * K + (col - Bc * K));
      } else {
        const int d = (int)(col - row);
        if (d < -g.s || d > g.r) return 0.0;
        return __ldg(g.data + g.boff[d + K] + row);
      }
    };
    if (tid < K) {
      double sg = 0.0, ab = 0.0;
      if (Pt.ls >= 0) {
        const long row = Pt.ls + tid;
        for (int t = 0; t < 2 * K && t < L; ++t) {
          const double pr = at(row, b + t) * smf[t];
          sg += pr;
          ab += fabs(pr);
        }
      }
      rc[tid] = sg;
      rc[K + tid] = ab;
    } else if (tid >= 16 && tid < 16 + K) {
      const int u = tid - 16;
      double sg = 0.0, ab = 0.0;
      if (Pt.rs >= 0) {
        const long row = Pt.rs + u;
        for (int t = 1; t <= 2 * K && t <= L; ++t) {
          const double pr = at(row, b + L - t) * smf[L - t];
          sg += pr;
          ab += fabs(pr);
        }
      }
      rc[2 * K + u] = sg;
      rc[3 * K + u] = ab;
    }
  }
}

// ---------------------------------------------------------------------------
// body solver, narrow variant (block tridiagonal): LPB lanes per body, MC
// block rows per lane, 32 / LPB bodies per warp.  Rows come straight from
// global memory (each lane reads its own contiguous block rows); the chunk
// state (AP, CP, DP per row) is parked in a lane-interleaved shared stash
// instead of registers; the interface system has LPB rows (log2 LPB block-PCR
// steps).  MC = 4: a quarter of the block-PCR work per block row of the
// 2-rows-per-lane kernel, 37 KB of stash per warp (config 2: 3.6x fewer
// instructions; ncu profiles/r01_*cfg2*).
// ---------------------------------------------------------------------------
template <int K, int MC, int LPB>
struct BlkNarrow {
  static constexpr int SR = 2 * K * K + K;           // stash doubles per row
  static constexpr int BYTES = 8 * 32 * MC * SR;     // per warp
};

template <int K, int MC, int LPB>
__global__ void __launch_bounds__(32) blk_body_narrow_kernel(BlkArgs g) {
  static_assert(MC >= 3, "the chunk elimination's row-0 step needs at least 3 rows per lane");
  static_assert(LPB >= 2 && LPB <= 32 && (LPB & (LPB - 1)) == 0, "lanes per body: power of two");
  constexpr int KK = K * K, SR = BlkNarrow<K, MC, LPB>::SR, G = 32 / LPB;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double stash[];
  const int lane = threadIdx.x, grp = lane / LPB, r = lane % LPB;
  const int seg = blockIdx.x * G + grp;
  const bool live = seg < g.nseg;
  const GPart Pt = g.part[live ? seg : g.nseg - 1];
  const long b = Pt.b;
  const int L = Pt.L, NB = L / K;
  const long B0 = b / K, NBall = g.n / K;
  const bool hasl = live && Pt.ls >= 0, hasr = live && Pt.rs >= 0;
  // the lane's block rows (and rhs) into L2 while the separator kernel runs:
  // the chunk elimination below reads them one block row at a time
  if (live) {
#pragma unroll
    for (int j = 0; j < MC; ++j) {
      const int q = r * MC + j;
      const long B = B0 + q;
      if (q < NB && B > 0) {
        const char* p0 = reinterpret_cast<const char*>(g.data + (3 * B - 1) * KK);
        for (int o = 0; o < 3 * KK * 8; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(g.f + b + (long)q * K));
      }
    }
  }
  Vec<K> xl, xrv;
  pdl_wait();     // separator values from the previous kernel
  pdl_trigger();  // the certificate kernel may launch (it waits for this grid before reading the records)
#pragma unroll
  for (int u = 0; u < K; ++u) {
    xl.v[u] = hasl ? __ldg(g.xsep + (long)(seg - 1) * K + u) : 0.0;
    xrv.v[u] = hasr ? __ldg(g.xsep + (long)seg * K + u) : 0.0;
  }
  auto st = [&](int j, int e) -> double& { return stash[(j * SR + e) * 32 + lane]; };
  auto put = [&](int j, const Blk<K>& A, const Blk<K>& C, const Vec<K>& D) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
#pragma unroll
      for (int v = 0; v < K; ++v) {
        st(j, u * K + v) = A.v[u][v];
        st(j, KK + u * K + v) = C.v[u][v];
      }
      st(j, 2 * KK + u) = D.v[u];
    }
  };
  auto get = [&](int j, Blk<K>& A, Blk<K>& C, Vec<K>& D) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
#pragma unroll
      for (int v = 0; v < K; ++v) {
        A.v[u][v] = st(j, u * K + v);
        C.v[u][v] = st(j, KK + u * K + v);
      }
      D.v[u] = st(j, 2 * KK + u);
    }
  };
  // block row q of the body: sub / diag / super block pointers (padding = identity,
  // separator couplings folded into the rhs)
  auto rowp = [&](int q) -> const double* {
    const long B = B0 + q;
    return g.data + (B == 0 ? -KK : (3 * B - 1) * KK);  // sub | diag | super
  };
  const bool vec = ((reinterpret_cast<uintptr_t>(g.data) | reinterpret_cast<uintptr_t>(g.f)) & 31) == 0;
  auto load_blk = [&](int q, int t, Blk<K>& X) {  // t = 0 sub, 1 diag, 2 super
    const long B = B0 + q;
    const bool pad = !live || q >= NB;
    const bool zero = t == 0 ? (q == 0 || B == 0) : (t == 2 ? (q == NB - 1 || B + 1 >= NBall) : false);
    const double* p = rowp(q) + t * KK;
    if constexpr (K == 4) {  // block rows of 4 x 32 B: one LDG.256 per block row (data / f 32-byte aligned)
      if (vec && !pad && !zero) {
#pragma unroll
        for (int u = 0; u < 4; ++u) ldg256(p + 4 * u, X.v[u][0], X.v[u][1], X.v[u][2], X.v[u][3]);
        return;
      }
    }
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int v = 0; v < K; ++v)
        X.v[u][v] = pad ? (t == 1 && u == v ? 1.0 : 0.0) : (zero ? 0.0 : __ldg(p + u * K + v));
  };
  auto load_f = [&](int q, Vec<K>& F) {
    const bool pad = !live || q >= NB;
    if constexpr (K == 4) {
      if (vec && !pad) ldg256(g.f + b + (long)q * K, F.v[0], F.v[1], F.v[2], F.v[3]);
    }
#pragma unroll
    for (int u = 0; u < K; ++u)
      if (!(K == 4 && vec && !pad)) F.v[u] = pad ? 0.0 : __ldg(g.f + b + (long)q * K + u);
    if (pad) return;
    if (q == 0 && hasl) {  // F -= A(first row, left separator) x_l
      const double* p = rowp(q);
#pragma unroll
      for (int u = 0; u < K; ++u)
#pragma unroll
        for (int v = 0; v < K; ++v) F.v[u] = fma(-__ldg(p + u * K + v), xl.v[v], F.v[u]);
    }
    if (q == NB - 1 && hasr) {  // F -= C(last row, right separator) x_r
      const double* p = rowp(q) + 2 * KK;
#pragma unroll
      for (int u = 0; u < K; ++u)
#pragma unroll
        for (int v = 0; v < K; ++v) F.v[u] = fma(-__ldg(p + u * K + v), xrv.v[v], F.v[u]);
    }
  };
  // ---- chunk elimination (Laszlo): AP_j y_first + y_j + CP_j y_last = DP_j, rows to the stash
  const int q0 = r * MC;
  double rsum = 0.0;
  Blk<K> APp, CPp;
  Vec<K> DPp;
#pragma unroll 1
  for (int j = 0; j < MC; ++j) {
    const int q = q0 + j;
    Blk<K> Ab, Db;
    load_blk(q, 0, Ab);
    load_blk(q, 1, Db);
    Vec<K> Fv;
    load_f(q, Fv);
    Blk<K> APj, CPj;
    Vec<K> DPj;
    if (j >= 2) blk_mul_sub<K>(Db, Ab, CPp);
    blk_inv<K>(Db, &rsum);
    if (j >= 2) blk_mv_sub<K>(Fv, Ab, DPp);
    DPj = blk_mv<K>(Db, Fv);
    if (j >= 2) {
      const Blk<K> aap = blk_mul<K>(Ab, APp);
      APj = blk_mul<K>(Db, aap);
      blk_neg<K>(APj);
    } else {
      APj = blk_mul<K>(Db, Ab);
    }
    {
      Blk<K> Cb;
      load_blk(q, 2, Cb);
      CPj = blk_mul<K>(Db, Cb);
    }
    put(j, APj, CPj, DPj);
    APp = APj;
    CPp = CPj;
    DPp = DPj;
  }
  // backward: rows MC-3 .. 1 in terms of (y_first, y_last)
  {
    Blk<K> An = APp, Cn = CPp;  // row j+1 (starts at MC-2 below)
    Vec<K> Dn = DPp;
    get(MC - 2, An, Cn, Dn);
#pragma unroll 1
    for (int j = MC - 3; j >= 1; --j) {
      Blk<K> Aj, Cj;
      Vec<K> Dj;
      get(j, Aj, Cj, Dj);
      blk_mv_sub<K>(Dj, Cj, Dn);
      blk_mul_sub<K>(Aj, Cj, An);
      Cj = blk_mul<K>(Cj, Cn);
      blk_neg<K>(Cj);
      put(j, Aj, Cj, Dj);
      An = Aj;
      Cn = Cj;
      Dn = Dj;
    }
  }
  // row 0 in terms of (y_prev_last, y_0, y_last)
  Blk<K> A0, C0;
  Vec<K> D0;
  get(0, A0, C0, D0);
  {
    Blk<K> A1, C1;
    Vec<K> D1;
    get(1, A1, C1, D1);
    Blk<K> R;
    blk_set_eye<K>(R);
    blk_mul_sub<K>(R, C0, A1);
    blk_inv<K>(R, &rsum);
    blk_mv_sub<K>(D0, C0, D1);
    D0 = blk_mv<K>(R, D0);
    A0 = blk_mul<K>(R, A0);
    const Blk<K> cc = blk_mul<K>(C0, C1);
    C0 = blk_mul<K>(R, cc);
    blk_neg<K>(C0);
    put(0, A0, C0, D0);
  }
  // ---- interface rows (LPB per body), block PCR inside the lane group;
  // row MC-1 (APp, CPp, DPp) is unchanged by the backward pass and stays in the stash
  Blk<K> al, ga, be;
  Vec<K> de = D0;
  blk_set_eye<K>(be);
  blk_set_zero<K>(al);
  {
    const int lo1 = r > 0 ? lane - 1 : lane;
    const Blk<K> pa = blk_shfl<K>(APp, lo1);
    const Blk<K> pc = blk_shfl<K>(CPp, lo1);
    const Vec<K> pd = vec_shfl<K>(DPp, lo1);
    if (r > 0) {
      al = blk_mul<K>(A0, pa);
      blk_neg<K>(al);
      blk_mul_sub<K>(be, A0, pc);
      blk_mv_sub<K>(de, A0, pd);
    }
  }
  blk_mul_sub<K>(be, C0, APp);
  blk_mv_sub<K>(de, C0, DPp);
  ga = blk_mul<K>(C0, CPp);
  blk_neg<K>(ga);
  blk_inv<K>(be, &rsum);
  al = blk_mul<K>(be, al);
  ga = blk_mul<K>(be, ga);
  de = blk_mv<K>(be, de);
  const bool jac = blk_jacobi<K>(al, ga, de, r, LPB);
#pragma unroll 1
  for (int sd = 1; sd < (jac ? 1 : LPB); sd <<= 1) {
    const bool hl = r >= sd, hh = r + sd < LPB;
    const int sl = hl ? lane - sd : lane, sh = hh ? lane + sd : lane;
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
    blk_inv<K>(nb, &rsum);
    al = blk_mul<K>(nb, na);
    blk_neg<K>(al);
    ga = blk_mul<K>(nb, ng);
    blk_neg<K>(ga);
    de = blk_mv<K>(nb, nd);
  }
  // ---- back-substitution, x straight to global
  const Vec<K> Fv = de;
  Vec<K> Fn = vec_shfl<K>(Fv, r + 1 < LPB ? lane + 1 : lane);
  if (r + 1 == LPB)
#pragma unroll
    for (int u = 0; u < K; ++u) Fn.v[u] = 0.0;
  Vec<K> Ev;
  {
    Blk<K> aE, cE;
    get(MC - 1, aE, cE, Ev);
    blk_mv_sub<K>(Ev, aE, Fv);
    blk_mv_sub<K>(Ev, cE, Fn);
  }
  bool finite = true;
  Vec<K> yfirst = Fv, ylast;
#pragma unroll
  for (int u = 0; u < K; ++u) ylast.v[u] = 0.0;
  const int qlast = NB - 1;
#pragma unroll 1
  for (int j = 0; j < MC; ++j) {
    Vec<K> y;
    if (j == 0) {
      y = Fv;
    } else if (j == MC - 1) {
      y = Ev;
    } else {
      Blk<K> Aj, Cj;
      Vec<K> Dj;
      get(j, Aj, Cj, Dj);
      y = Dj;
      blk_mv_sub<K>(y, Aj, Fv);
      blk_mv_sub<K>(y, Cj, Ev);
    }
    const int q = q0 + j;
    if (live && q < NB) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        finite &= isfinite(y.v[u]);
        g.x[b + (long)q * K + u] = y.v[u];
      }
      if (q == qlast) ylast = y;
    }
  }
  if (live && r == 0 && hasr)
#pragma unroll
    for (int u = 0; u < K; ++u) g.x[Pt.rs + u] = xrv.v[u];
  if (g.status) {
    const unsigned gm = (LPB == 32 ? FULL : ((1u << LPB) - 1u)) << (grp * LPB);
    const unsigned badp = __ballot_sync(FULL, !isfinite(rsum)) & gm;
    const unsigned badf = __ballot_sync(FULL, !finite) & gm;
    if (live && r == 0) {
      if (badp) status_pivot(g.status, seg);
      if (badf) status_nonfinite(g.status, seg);
    }
  }
  // ---- certificate records: separator rows' couplings to the first / last body block
  if (g.rec && live) {
    double* rc = g.rec + (long)seg * 4 * K;
    if (r == 0) {  // left: the separator block row's super block times y(first block)
#pragma unroll
      for (int u = 0; u < K; ++u) {
        double sg = 0.0, ab = 0.0;
        if (hasl) {
          const long BS = B0 - 1;
          const double* cp = g.data + (BS == 0 ? KK : (3 * BS - 1) * KK + 2 * KK);
#pragma unroll
          for (int v = 0; v < K; ++v) {
            const double pr = __ldg(cp + u * K + v) * yfirst.v[v];
            sg += pr;
            ab += fabs(pr);
          }
        }
        rc[u] = sg;
        rc[K + u] = ab;
      }
    }
    if (q0 <= qlast && qlast < q0 + MC) {  // right: its sub block times y(last block)
#pragma unroll
      for (int u = 0; u < K; ++u) {
        double sg = 0.0, ab = 0.0;
        if (hasr) {
          const long BR = B0 + NB;
          const double* ap = g.data + (3 * BR - 1) * KK;
#pragma unroll
          for (int v = 0; v < K; ++v) {
            const double pr = __ldg(ap + u * K + v) * ylast.v[v];
            sg += pr;
            ab += fabs(pr);
          }
        }
        rc[2 * K + u] = sg;
        rc[3 * K + u] = ab;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// speculative factor: warp per separator, half-warp per side, one block
// element per lane (lane e = 4u + v of its half), HB block rows per side.
// ---------------------------------------------------------------------------
struct BlkSpecArgs {
  const double* data;
  long n;
  int s, r;
  int layout;
  int nsep;
  const int* sep;  // separator start rows
  const double* f; // right-hand side
  double* xsep;    // out: per separator its K values
  double* Tdiag;   // out: per separator the K*K block A_SS (certificate)
  DevStatus* reset;  // the solve's status slot (reset by block 0)
  long boff[9];    // banded: A(row, row + d) = data[boff[d + K] + row]
  long data_len;   // entries in data (staging over-read bound)
};

// A(i, j) for the block kinds (0 outside the structure)
__device__ __forceinline__ double blk_at(const BlkSpecArgs& g, int K, long i, long j) {
  if (i < 0 || j < 0 || i >= g.n || j >= g.n) return 0.0;
  if (g.layout == kBlkBlockTri) {
    const long bi = i / K, bj = j / K;
    if (bi - bj > 1 || bj - bi > 1) return 0.0;
    const long off = bi == 0 ? 0 : (3 * bi - 1) * (long)K * K;
    const long blk = bi > 0 ? bj - bi + 1 : bj - bi;
    return __ldg(g.data + off + blk * K * K + (i - bi * K) * K + (j - bj * K));
  }
  const long d = j - i;
  if (d < -g.s || d > g.r) return 0.0;
  return __ldg(g.data + g.boff[d + K] + i);
}

// distributed K x K (K <= 4) algebra inside a 16-lane half (base 0 or 16),
// lane base + 4u + v holds element (u, v); lanes with u or v >= K hold 0.
__device__ __forceinline__ double dmul(double a, double b, int base, int u, int v, int K) {
  double acc = 0.0;
  for (int l = 0; l < K; ++l)
    acc = fma(__shfl_sync(0xffffffffu, a, base + u * 4 + l), __shfl_sync(0xffffffffu, b, base + l * 4 + v), acc);
  return acc;
}
// the same product with the left operand already held as row u in every
// lane of that row (no shuffles for it): acc = sum_l arow[l] B(l, v)
__device__ __forceinline__ double dmul_row(const double (&arow)[4], double b, int base, int v, int K) {
  double acc = 0.0;
  for (int l = 0; l < K; ++l) acc = fma(arow[l], __shfl_sync(0xffffffffu, b, base + l * 4 + v), acc);
  return acc;
}
// in-place Gauss-Jordan inverse without pivoting
__device__ __forceinline__ double dinv(double a, int base, int u, int v, int K, double* rsum) {
  for (int k = 0; k < K; ++k) {
    const double akk = __shfl_sync(0xffffffffu, a, base + k * 4 + k);
    const double auk = __shfl_sync(0xffffffffu, a, base + u * 4 + k);
    const double akv = __shfl_sync(0xffffffffu, a, base + k * 4 + v);
    const double p = fast_rcp(akk);
    if (u == 0 && v == 0) *rsum += fabs(p);
    if (u == k && v == k)
      a = p;
    else if (u == k)
      a = akv * p;
    else if (v == k)
      a = -auk * p;
    else
      a = fma(-auk * p, akv, a);
  }
  return a;
}

template <int K, int HB, int NS = 2>
__global__ void __launch_bounds__(128) blk_spec_fused_kernel(BlkSpecArgs g) {
  pdl_trigger();  // the body kernel may launch and stage its rows early
  const int lane = threadIdx.x & 31;
  const int j0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NS;
  if (g.reset && blockIdx.x == 0 && threadIdx.x < kCertSlots + 2) {  // first kernel of the solve: fresh status
    if (threadIdx.x < kCertSlots)
      g.reset->cert_bits[threadIdx.x] = 0ull;
    else if (threadIdx.x == kCertSlots)
      g.reset->bad_seg = INT_MAX;
    else
      g.reset->pivot_seg = INT_MAX;
  }
  if (j0 >= g.nsep) return;  // warp-uniform
  constexpr int KK = K * K;
  const int h = lane >> 4, e = lane & 15, u = e >> 2, v = e & 3;
  const int base = h << 4;
  const bool act = u < K && v < K;
  const bool vec = u < K && v == 0;  // block vectors live in column 0
  const double eye = (u == v) ? 1.0 : 0.0;
  const long n = g.n;
  // NS separators per warp, their block chains interleaved (independent
  // shuffle / FP64 dependency chains in flight together).  Both halves run
  // the same far -> near elimination (no divergence around the shuffles).
  // Block i = 0 (far) .. HB-1 (near) of side h starts at row
  //   trailing (h = 0): S - (HB - i) K      leading (h = 1): S + K + (HB - 1 - i) K
  // and couples to its farther neighbour through Fc (trailing: sub, leading:
  // super) and to its nearer neighbour through Nc.  Element (u, v) of the
  // sub / diag / super block of the block row at r0: t = 0 / 1 / 2.
  const int tF = h == 0 ? 0 : 2, tN = 2 - tF;
  auto prep = [&](int t, long& off, bool& ok) {
    const int d = v - u + (t - 1) * K;
    ok = act && (g.layout == kBlkBlockTri || (d >= -g.s && d <= g.r));
    off = g.layout == kBlkBlockTri ? (long)t * KK + u * K + v : (ok ? g.boff[d + K] + u : 0);
  };
  long oD, oF, oN;
  bool kD, kF, kN;
  prep(1, oD, kD);
  prep(tF, oF, kF);
  prep(tN, oN, kN);
  auto ld = [&](long r0, int t, long off, bool ok) -> double {
    if (!ok) return 0.0;
    if (g.layout == kBlkBlockTri) {
      const long B = r0 / K;
      return (B + t - 1 >= 0 && B + t - 1 < n / K) ? __ldg(g.data + (3 * B - 1) * KK + off) : 0.0;
    }
    const long col = r0 + v + (t - 1) * K;
    return (col >= 0 && col < n) ? __ldg(g.data + off + r0) : 0.0;
  };
  auto ldf = [&](long r0) -> double { return vec ? __ldg(g.f + r0 + u) : 0.0; };
  long S[NS];
  double Bc[NS], Cc[NS], Dss[NS], fS[NS], Dn[NS], Fn[NS], Nn[NS], fn[NS], G[NS], Ncp[NS], y[NS];
  auto row0 = [&](int q, int i) -> long {
    return h == 0 ? S[q] - (long)(HB - i) * K : S[q] + K + (long)(HB - 1 - i) * K;
  };
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    S[q] = g.sep[min(j0 + q, g.nsep - 1)];
    // couplings with the separator: B1 = A(S+u, S-K+v) / C0 = A(S+u, S+K+v);
    // near block -> separator: A(S-K+u, S+v) / A(S+K+u, S+v)
    Bc[q] = act ? blk_at(g, K, S[q] + u, h == 0 ? S[q] - K + v : S[q] + K + v) : 0.0;
    Cc[q] = act ? blk_at(g, K, h == 0 ? S[q] - K + u : S[q] + K + u, S[q] + v) : 0.0;
    Dss[q] = act ? blk_at(g, K, S[q] + u, S[q] + v) : eye;
    fS[q] = ldf(S[q]);
    const long r = row0(q, 0);
    Dn[q] = act ? ld(r, 1, oD, kD) : eye;
    Fn[q] = ld(r, tF, oF, kF);
    Nn[q] = ld(r, tN, oN, kN);
    fn[q] = ldf(r);
    G[q] = Ncp[q] = y[q] = 0.0;
  }
  double rsum = 0.0;
  // far -> near sweep with the next block's loads in flight:
  //   D'_i = D_i - Fc_i G_{i-1} Nc_{i-1},  G_i = D'_i^-1,  y_i = f_i - Fc_i G_{i-1} y_{i-1}
#pragma unroll
  for (int i = 0; i < HB; ++i) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      double D = Dn[q];
      const double Fc = Fn[q], Nc = Nn[q], fi = fn[q];
      if (i + 1 < HB) {
        const long r1 = row0(q, i + 1);
        Dn[q] = act ? ld(r1, 1, oD, kD) : eye;
        Fn[q] = ld(r1, tF, oF, kF);
        Nn[q] = ld(r1, tN, oN, kN);
        fn[q] = ldf(r1);
      }
      if (i > 0) {
        // Fc is the left operand of both products: its row u gathered once
        double frow[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) frow[l] = l < K ? __shfl_sync(0xffffffffu, Fc, base + u * 4 + l) : 0.0;
        D -= dmul_row(frow, dmul(G[q], Ncp[q], base, u, v, K), base, v, K);
        y[q] = fi - dmul_row(frow, dmul(G[q], y[q], base, u, v, K), base, v, K);
      } else {
        y[q] = fi;
      }
      const double Gi = dinv(D, base, u, v, K, &rsum);
      G[q] = act ? Gi : 0.0;
      Ncp[q] = Nc;
    }
  }
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    // near diagonal block of the truncated inverse Xn = G: this side's Schur
    // term B Xn C and condensed rhs B Xn y
    const double part = dmul(Bc[q], dmul(G[q], Cc[q], base, u, v, K), base, u, v, K);
    const double rpart = dmul(Bc[q], dmul(G[q], y[q], base, u, v, K), base, u, v, K);
    const double other = __shfl_xor_sync(0xffffffffu, part, 16);
    const double rother = __shfl_xor_sync(0xffffffffu, rpart, 16);
    double Ti = dinv(Dss[q] - part - other, base, u, v, K, &rsum);
    if (!act) Ti = 0.0;
    const double rhs = vec ? (fS[q] - rpart) - rother : 0.0;
    const double xs = dmul(Ti, rhs, base, u, v, K);
    const int j = j0 + q;
    if (j < g.nsep) {
      if (h == 0 && act) g.Tdiag[(long)j * KK + u * K + v] = Dss[q];
      if (h == 0 && vec) g.xsep[(long)j * K + u] = xs;
    }
  }
  (void)rsum;  // a vanished pivot leaves non-finite separator values: the certificate rejects them
}

// K x K block at p (row-major) into registers: 256-bit loads for K = 4 / 2 when
// the data is 32-byte aligned
template <int K>
__device__ __forceinline__ void blktri_ld(const double* p, bool vec, Blk<K>& X, unsigned long long pol = 0) {
  if constexpr (K == 4) {
    if (vec) {
      if (pol) {
#pragma unroll
        for (int u = 0; u < 4; ++u) ldg256h(p + 4 * u, pol, X.v[u][0], X.v[u][1], X.v[u][2], X.v[u][3]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) ldg256(p + 4 * u, X.v[u][0], X.v[u][1], X.v[u][2], X.v[u][3]);
      }
      return;
    }
  } else if constexpr (K == 2) {
    if (vec) {
      ldg256(p, X.v[0][0], X.v[0][1], X.v[1][0], X.v[1][1]);
      return;
    }
  }
#pragma unroll
  for (int u = 0; u < K; ++u)
#pragma unroll
    for (int v = 0; v < K; ++v) X.v[u][v] = __ldg(p + u * K + v);
}

// ---------------------------------------------------------------------------
// body solver, block tridiagonal, TWO THREADS PER BODY (blktri_body_kernel):
// exact given the separators.  The top thread eliminates block rows 0..m-1
// top-down (block Thomas / LU without pivoting, src/localfact.cpp:84-100),
//   D'_i = D_i - A_i G_{i-1},  G_i = D'_i^-1 C_i,  z_i = D'_i^-1 (f_i - A_i z_{i-1}),
// the bottom thread block rows NB-1..m bottom-up (the mirror image, UL),
//   D''_i = D_i - C_i H_{i+1}, H_i = D''_i^-1 A_i, w_i = D''_i^-1 (f_i - C_i w_{i+1});
// they meet at rows m-1 / m: (I - G_{m-1} H_m) x_{m-1} = z_{m-1} - G_{m-1} w_m,
// x_m = w_m - H_m x_{m-1}, and back-substitute outwards from the (G, z) / (H, w)
// they parked in a global scratch (one 20-double record per block row, written
// and read by the same thread moments apart: mostly L2).  Block rows arrive by
// 256-bit loads (K = 4, aligned data; an L2 prefetch 4 block rows ahead or an
// L1 prefetch of the next one measured no better or worse).
// No shared memory beyond the 2 x 32 meeting records: every body of config 2
// is in flight at once (2 threads x 16384 bodies), and there is no lane-level
// reduced system at all.  The separator couplings of the first / last block
// rows are folded into f.  CTA = 2 warps over 32 bodies: warp 0 the top
// halves, warp 1 the bottom halves.
// ---------------------------------------------------------------------------
template <int K, int H>
__device__ __forceinline__ void blktri_half(const BlkArgs& g, double* scr, bool live, int seg, const GPart& Pt,
                                            Blk<K>& Gm, Vec<K>& zm, double& rsum) {
  constexpr int KK = K * K, SR = KK + K;
  const long b = Pt.b;
  const int NB = Pt.L / K, m = NB / 2;
  const long B0 = b / K, NBall = g.n / K;
  const bool vec = ((reinterpret_cast<uintptr_t>(g.data) | reinterpret_cast<uintptr_t>(g.f) |
                     reinterpret_cast<uintptr_t>(scr)) & 31) == 0;
  const int i0 = H == 0 ? 0 : NB - 1, cnt = H == 0 ? m : NB - m;
  auto rowB = [&](int s) -> long { return B0 + (H == 0 ? i0 + s : i0 - s); };
  pdl_wait();  // separator values from the separator kernel
  Vec<K> xs;   // this half's outer separator (top: left, bottom: right)
  const bool hs = live && (H == 0 ? Pt.ls >= 0 : Pt.rs >= 0);
#pragma unroll
  for (int u = 0; u < K; ++u) xs.v[u] = hs ? __ldg(g.xsep + (long)(H == 0 ? seg - 1 : seg) * K + u) : 0.0;
  // L2: the rows stream through once (evict_first); the parked records come
  // back within the same body sweep (evict_last: keep them out of DRAM)
  const unsigned long long pin = l2_evict_first(), pkeep = l2_evict_last();
  Blk<K> P;  // previous step's G (top) / H (bottom)
  Vec<K> q;  // previous step's z / w
  blk_set_zero<K>(P);
#pragma unroll
  for (int u = 0; u < K; ++u) q.v[u] = 0.0;
#pragma unroll 1
  for (int s = 0; s < (live ? cnt : 0); ++s) {
    const long B = rowB(s);
    const double* p = g.data + (3 * B - 1) * KK;  // sub | diag | super (B >= 1 unless s == 0 at the top)
    Blk<K> Fc, D, Nc;  // coupling to the previous step's row (F), toward the meeting point (N)
    Vec<K> y;
    const bool first = B == 0;  // block row 0 of the matrix: [diag | super] at 0
    const double* pd = first ? g.data : p + KK;
    blktri_ld<K>(pd, vec, D, pin);
    const bool hasF = H == 0 ? B > 0 : B + 1 < NBall;  // the far coupling block exists
    const bool hasN = H == 0 ? B + 1 < NBall : B > 0;
    if (hasF) blktri_ld<K>(H == 0 ? p : p + 2 * KK, vec, Fc, pin); else blk_set_zero<K>(Fc);
    if (hasN) blktri_ld<K>(H == 0 ? pd + KK : p, vec, Nc, pin); else blk_set_zero<K>(Nc);
    if (K == 4 && vec) {
      ldg256h(g.f + B * K, pin, y.v[0], y.v[1], y.v[2], y.v[3]);
    } else {
#pragma unroll
      for (int u = 0; u < K; ++u) y.v[u] = __ldg(g.f + B * K + u);
    }
    if (s == 0) {  // the outer separator's coupling to the rhs
      if (hs) blk_mv_sub<K>(y, Fc, xs);
    } else {
      blk_mul_sub<K>(D, Fc, P);
      blk_mv_sub<K>(y, Fc, q);
    }
    blk_inv<K>(D, &rsum);
    P = blk_mul<K>(D, Nc);
    q = blk_mv<K>(D, y);
    if (s + 1 < cnt) {  // park (G, z) / (H, w) for the back-substitution
      double* r = scr + B * SR;
      if (K == 4 && vec) {  // 160-byte records, 32-byte aligned: five 256-bit stores
#pragma unroll
        for (int u = 0; u < K; ++u) stg256h(r + 4 * u, pkeep, P.v[u][0], P.v[u][1 % K], P.v[u][2 % K], P.v[u][3 % K]);
        stg256h(r + KK, pkeep, q.v[0], q.v[1 % K], q.v[2 % K], q.v[3 % K]);
      } else {
#pragma unroll
        for (int u = 0; u < K; ++u) {
#pragma unroll
          for (int v = 0; v < K; ++v) r[u * K + v] = P.v[u][v];
          r[KK + u] = q.v[u];
        }
      }
    }
  }
  Gm = P;
  zm = q;
}

template <int K, int H>
__device__ __forceinline__ void blktri_back(const BlkArgs& g, const double* scr, bool live, const GPart& Pt,
                                            Vec<K> x, bool& finite) {
  constexpr int KK = K * K, SR = KK + K;
  const long b = Pt.b;
  const int NB = Pt.L / K, m = NB / 2;
  const long B0 = b / K;
  const bool vec = ((reinterpret_cast<uintptr_t>(g.x) | reinterpret_cast<uintptr_t>(scr)) & 31) == 0;
  const unsigned long long pgone = l2_evict_first();  // parked records: last use; x: streamed out
  // x holds the meeting row's value (top: m-1, bottom: m); walk outwards
  const int i0 = H == 0 ? m - 1 : m, cnt = H == 0 ? m : NB - m;
#pragma unroll 1
  for (int s = 0; s < (live ? cnt : 0); ++s) {
    const long B = B0 + (H == 0 ? i0 - s : i0 + s);
    if (s > 0) {
      const double* r = scr + B * SR;
      Blk<K> Pr;
      Vec<K> y;
      if (K == 4 && vec) {
#pragma unroll
        for (int u = 0; u < K; ++u) ldg256h(r + 4 * u, pgone, Pr.v[u][0], Pr.v[u][1 % K], Pr.v[u][2 % K], Pr.v[u][3 % K]);
        ldg256h(r + KK, pgone, y.v[0], y.v[1 % K], y.v[2 % K], y.v[3 % K]);
      } else {
#pragma unroll
        for (int u = 0; u < K; ++u) {
          y.v[u] = r[KK + u];
#pragma unroll
          for (int v = 0; v < K; ++v) Pr.v[u][v] = r[u * K + v];
        }
      }
      blk_mv_sub<K>(y, Pr, x);
      x = y;
    }
#pragma unroll
    for (int u = 0; u < K; ++u) finite &= isfinite(x.v[u]);
    if (K == 4 && vec)
      stg256h(g.x + B * K, pgone, x.v[0], x.v[1 % K], x.v[2 % K], x.v[3 % K]);
    else
#pragma unroll
      for (int u = 0; u < K; ++u) g.x[B * K + u] = x.v[u];
  }
}

template <int K>
__global__ void __launch_bounds__(64) blktri_body_kernel(BlkArgs g, double* scr) {
  constexpr int KK = K * K;
  __shared__ double meet[32][KK + K];
  const int tid = threadIdx.x, lane = tid & 31, h = tid >> 5;
  const int seg = blockIdx.x * 32 + lane;
  const bool live = seg < g.nseg;
  const GPart Pt = g.part[live ? seg : g.nseg - 1];
  pdl_trigger();  // the certificate kernel may launch (it waits for this grid)
  double rsum = 0.0;
  Blk<K> Gm;
  Vec<K> zm;
  if (h == 0)
    blktri_half<K, 0>(g, scr, live, seg, Pt, Gm, zm, rsum);
  else
    blktri_half<K, 1>(g, scr, live, seg, Pt, Gm, zm, rsum);
  if (h == 1) {  // (H_m, w_m) to the top thread
#pragma unroll
    for (int u = 0; u < K; ++u) {
      meet[lane][KK + u] = zm.v[u];
#pragma unroll
      for (int v = 0; v < K; ++v) meet[lane][u * K + v] = Gm.v[u][v];
    }
  }
  __syncthreads();
  Vec<K> xm;
  if (h == 0) {  // (I - G_{m-1} H_m) x_{m-1} = z_{m-1} - G_{m-1} w_m
    Blk<K> Hm, M;
    Vec<K> wm;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      wm.v[u] = meet[lane][KK + u];
#pragma unroll
      for (int v = 0; v < K; ++v) Hm.v[u][v] = meet[lane][u * K + v];
    }
    blk_set_eye<K>(M);
    blk_mul_sub<K>(M, Gm, Hm);
    blk_inv<K>(M, &rsum);
    Vec<K> rhs = zm;
    blk_mv_sub<K>(rhs, Gm, wm);
    xm = blk_mv<K>(M, rhs);
  }
  __syncthreads();
  if (h == 0)
#pragma unroll
    for (int u = 0; u < K; ++u) meet[lane][u] = xm.v[u];
  __syncthreads();
  if (h == 1) {  // x_m = w_m - H_m x_{m-1}
    Vec<K> xt;
#pragma unroll
    for (int u = 0; u < K; ++u) xt.v[u] = meet[lane][u];
    xm = zm;
    blk_mv_sub<K>(xm, Gm, xt);
  }
  bool finite = true;
  if (h == 0)
    blktri_back<K, 0>(g, scr, live, Pt, xm, finite);
  else
    blktri_back<K, 1>(g, scr, live, Pt, xm, finite);
  if (g.status && live) {
    if (!isfinite(rsum)) status_pivot(g.status, seg);
    if (!finite) status_nonfinite(g.status, seg);
  }
  if (!live) return;
  const long B0 = Pt.b / K;
  const int NB = Pt.L / K;
  if (h == 1 && Pt.rs >= 0)
#pragma unroll
    for (int u = 0; u < K; ++u) g.x[Pt.rs + u] = __ldg(g.xsep + (long)seg * K + u);
  // certificate records (blk_cert_kernel format): the separator block rows'
  // couplings to this body's first (left) / last (right) block row
  if (g.rec) {
    double* rc = g.rec + (long)seg * 4 * K;
    const bool has = h == 0 ? Pt.ls >= 0 : Pt.rs >= 0;
    const long BB = h == 0 ? B0 : B0 + NB - 1;  // this body's boundary block row
    Vec<K> y;
#pragma unroll
    for (int u = 0; u < K; ++u) y.v[u] = g.x[BB * K + u];  // written by this thread above
    const double* cp = nullptr;
    if (has) {
      const long BS = h == 0 ? B0 - 1 : B0 + NB;  // the separator block row
      cp = h == 0 ? g.data + (BS == 0 ? KK : (3 * BS - 1) * KK + 2 * KK) : g.data + (3 * BS - 1) * KK;
    }
#pragma unroll
    for (int u = 0; u < K; ++u) {
      double sg = 0.0, ab = 0.0;
      if (has)
#pragma unroll
        for (int v = 0; v < K; ++v) {
          const double pr = __ldg(cp + u * K + v) * y.v[v];
          sg += pr;
          ab += fabs(pr);
        }
      rc[(h == 0 ? 0 : 2 * K) + u] = sg;
      rc[(h == 0 ? K : 3 * K) + u] = ab;
    }
  }
}

// ---------------------------------------------------------------------------
// speculative factor, block tridiagonal, ONE THREAD PER SEPARATOR SIDE with the
// K x K algebra in registers (blktri_spec_kernel).  The side's HB block rows
// stream straight from memory, one block row per step; K = 4 / 2 block
// rows are 128 / 32-byte multiples, read by 256-bit loads (one sector per
// request: the lanes of a warp walk different bodies, so the requests do not
// coalesce and the sector count is what the L1 pays for).  Far -> near block
// elimination (src/localfact.cpp:84-100 order):
//   D'_i = D_i - F_i X_{i-1},  X_i = D'_i^-1 N_i,  z_i = D'_i^-1 (f_i - F_i z_{i-1})
// with F the coupling away from the separator, N toward it; the near block row
// then is x_near = z_n - X_n x_S, and the separator block row gives
//   (A_SS - A_S,above X_above - C_S,below X_below) x_S = f_S - A_S,above z_above - C_S,below z_below.
// CTA = 2 warps over 32 separators: warp 0 the sides above, warp 1 below.
// ---------------------------------------------------------------------------
template <int K, int HB, int H>
__device__ __forceinline__ void blktri_side(const BlkSpecArgs& g, bool live, long BS, Blk<K>& T, Vec<K>& rr) {
  constexpr int KK = K * K;
  const long NBall = g.n / K;
  const bool vec = ((reinterpret_cast<uintptr_t>(g.data) | reinterpret_cast<uintptr_t>(g.f)) & 31) == 0;
  // block row Bi of step i (far -> near): H = 0: BS - HB + i, H = 1: BS + HB - i
  auto brow = [&](int i) -> long { return H == 0 ? BS - HB + i : BS + HB - i; };
  const bool ok = live && BS - HB >= 0 && BS + HB < NBall;  // the window inside the matrix
  struct Row {
    Blk<K> F, D, N;
    Vec<K> f;
  };
  auto load = [&](int i, Row& R) {
    const long B = ok ? brow(i) : 1;
    const double* p = g.data + (3 * B - 1) * KK;  // sub | diag | super (block row 0: diag | super at 0)
    // the far coupling of the farthest block row is dropped by the truncation
    // (and absent at the matrix ends): not read
    if (i > 0)
      blktri_ld<K>(p + (H == 0 ? 0 : 2 * KK), vec, R.F);
    else
      blk_set_zero<K>(R.F);
    blktri_ld<K>(p + KK, vec, R.D);
    blktri_ld<K>(p + (H == 0 ? 2 * KK : 0), vec, R.N);
    if (K == 4 && vec) {
      ldg256(g.f + B * K, R.f.v[0], R.f.v[1], R.f.v[2], R.f.v[3]);
    } else {
#pragma unroll
      for (int u = 0; u < K; ++u) R.f.v[u] = __ldg(g.f + B * K + u);
    }
  };
  Row cur;
  Blk<K> X;
  Vec<K> z;
  blk_set_zero<K>(X);
#pragma unroll
  for (int u = 0; u < K; ++u) z.v[u] = 0.0;
  double rsum = 0.0;
#pragma unroll 1
  for (int i = 0; i < HB; ++i) {
    load(i, cur);
    Blk<K> D = cur.D;
    Vec<K> y = cur.f;
    if (i > 0) {  // step 0: the truncation drops the coupling to the far side
      blk_mul_sub<K>(D, cur.F, X);
      blk_mv_sub<K>(y, cur.F, z);
    }
    blk_inv<K>(D, &rsum);
    X = blk_mul<K>(D, cur.N);
    z = blk_mv<K>(D, y);
  }
  // the separator block row's coupling to this side's near block row
  const double* ps = g.data + (3 * (ok ? BS : 1) - 1) * KK;
  Blk<K> As;
  blktri_ld<K>(ps + (H == 0 ? 0 : 2 * KK), vec, As);
  T = blk_mul<K>(As, X);
  rr = blk_mv<K>(As, z);
  if (!ok || !isfinite(rsum))
#pragma unroll
    for (int u = 0; u < K; ++u) rr.v[u] = __longlong_as_double(0x7ff8000000000000ll);
}

template <int K, int HB>
__global__ void __launch_bounds__(64) blktri_spec_kernel(BlkSpecArgs g) {
  constexpr int KK = K * K;
  __shared__ double xch[32][KK + K];
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
  pdl_trigger();  // the body kernel may launch and start loading
  const int lane = tid & 31, h = tid >> 5;
  const int j = blockIdx.x * 32 + lane;
  const bool live = j < g.nsep;
  const long BS = live ? g.sep[j] / K : 0;
  Blk<K> T;
  Vec<K> rr;
  if (h == 0)
    blktri_side<K, HB, 0>(g, live, BS, T, rr);
  else
    blktri_side<K, HB, 1>(g, live, BS, T, rr);
  if (h == 1) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
      xch[lane][KK + u] = rr.v[u];
#pragma unroll
      for (int v = 0; v < K; ++v) xch[lane][u * K + v] = T.v[u][v];
    }
  }
  __syncthreads();
  if (h == 0 && live) {
    const double* ps = g.data + (3 * BS - 1) * KK;
    Blk<K> A;
    Vec<K> rhs;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      rhs.v[u] = (__ldg(g.f + BS * K + u) - rr.v[u]) - xch[lane][KK + u];
#pragma unroll
      for (int v = 0; v < K; ++v) {
        const double ass = __ldg(ps + KK + u * K + v);
        A.v[u][v] = (ass - T.v[u][v]) - xch[lane][u * K + v];
        g.Tdiag[(long)j * KK + u * K + v] = ass;
      }
    }
    double rsum = 0.0;
    blk_inv<K>(A, &rsum);
    const Vec<K> xs = blk_mv<K>(A, rhs);
#pragma unroll
    for (int u = 0; u < K; ++u) g.xsep[(long)j * K + u] = xs.v[u];
  }
  // a vanished pivot leaves non-finite separator values: the certificate rejects them
}

// omega = max over separator rows of |f - A_SS x_S - left - right| / (|f| + sum |terms|).
template <int K>
__global__ void blk_cert_kernel(const double* __restrict__ Tdiag, const int* __restrict__ sep, int nsep,
                                const double* __restrict__ f, const double* __restrict__ xsep,
                                const double* __restrict__ rec, DevStatus* st, DevStatus* host_out,
                                unsigned* done_ctr) {
  pdl_wait();
  double worst = 0.0;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)nsep * K; t += (long)gridDim.x * blockDim.x) {
    const long j = t / K;
    const int u = (int)(t % K);
    const long S = sep[j];
    double sg = 0.0, ab = 0.0;
#pragma unroll
    for (int v = 0; v < K; ++v) {
      const double pr = Tdiag[j * K * K + u * K + v] * xsep[j * K + v];
      sg += pr;
      ab += fabs(pr);
    }
    const double* rl = rec + j * 4 * K;        // body j: its right separator is j
    const double* rr = rec + (j + 1) * 4 * K;  // body j+1: its left separator is j
    sg += rl[2 * K + u] + rr[u];
    ab += rl[3 * K + u] + rr[K + u];
    const double fv = f[S + u];
    const double num = fabs(fv - sg), den = fabs(fv) + ab;
    double om = den > 0 ? num / den : num;
    if (!(om <= 1.0e308)) om = __longlong_as_double(0x7ff0000000000000ll);
    worst = fmax(worst, om);
  }
  for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
  if ((threadIdx.x & 31) == 0 && worst > 0) status_cert(st, worst);
  if (host_out) status_publish_last(st, host_out, done_ctr);  // pinned host slot: no copy in the stream
}

}  // namespace psg
