// psg_local.cu -- per-partition local factorizations on the device: the
// reference's LocalFactorization (proj/include/parsol/localfact.hpp:24-125,
// src/localfact.cpp) behind the C ABI psg_local_* (include/psg.h), plus the
// dense reduced-system solve of solve_reduced(const ReducedSystem&)
// (src/parfact.cpp:134-184) as psg_dense_solve.
//
// The solver's hot path never builds these objects (its kernels work on the
// matrix in place, psg_capi.cu); they exist so that the reference's
// per-partition API -- factor(), factor_lu/lud/cyclic_reduction,
// factor_lu_pivot/qr, condense, backsolve, apply_N_inv/S_inv -- is a drop-in
// that runs on the GPU.  One CTA owns one partition block; the block's
// arrays live in one device arena.  Every update is issued in the
// reference's operation order and this translation unit is compiled with
// --fmad=false, so the results are bit-identical to the reference
// (tests/cpp/test_localfact.cpp, tests/test_localfact_gpu.py).
//
// Parallelism inside a CTA follows the data independence of each step:
//   banded LU   -- the (es x er) update rectangle of pivot k,
//   fill-ins    -- one thread per column of z, y, w, v,
//   products    -- one thread per entry of alpha/beta/gamma (k ascending),
//   CR          -- one thread per entry of each g x g block product,
//   dense frame -- rows of W/Lmat in parallel for a row operation, rows of
//                  Linv for the accumulated column update, pivot search by a
//                  CTA argmax (ties to the lowest row, as the serial scan).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/psg.h"

namespace {

constexpr int kThreads = 256;

struct LfFail {
  int code;
  std::string msg;
};

#define LF_TRY(expr)                                                                        \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) throw LfFail{PSG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
  } while (0)

int lf_err(char* err, size_t errlen, int code, const std::string& msg) {
  if (err && errlen) std::snprintf(err, errlen, "%s", msg.c_str());
  return 1 + code;
}

// status words written by the kernels
enum : int {
  ST_CODE = 0,    // 0 ok, else 1 + psg_errc
  ST_DETAIL = 1,  // body row of a zero pivot
  ST_NAORD = 2,   // dense: retired pivots
  ST_NDEF = 3,    // dense: deferred pivots (extras)
  ST_NELIM = 4,   // CR: eliminations
  ST_LEVELS = 5,  // CR: reduction levels
  ST_NREM = 6,    // CR: remaining block rows (1 or 2)
  ST_REM0 = 7,
  ST_REM1 = 8,
  ST_COUNT = 16
};

// Device view of one partition block and every array its factorization
// produces (pointers into one arena; unused ones are null).
struct LfDev {
  int strategy, L, k0, k1, es, er, kind, m, s, r;
  double tol;
  // inputs (PartitionBlock)
  const double *env, *b0, *c0, *b1, *c1, *ar;
  // outputs common to every core
  double *z, *w, *y, *v, *a1, *a2, *be, *ga, *kept;
  // banded core
  double *fac, *dvec, *mu;
  int* flag;
  // cyclic core
  int g, nb;
  double *ca, *cd, *cc;  // working a / d / c blocks, nb each
  int *elim_idx, *act, *keep;
  double* elim_mat;  // per elimination: ml, mr, a, c, dinv (g x g each)
  double *d2, *d2inv, *cmat, *rmat, *rmd2, *corr, *tmp, *lu;
  int* perm;
  // dense recorded core
  int dim;
  double *W, *Lm, *Li, *vv;
  int *row_state, *col_state, *a_order, *deferred, *kept_rows, *kept_cols, *pair_row, *ext_pos;
  double* ext_alpha;
  int* st;
};

__device__ __forceinline__ double body_at(const LfDev& d, int i, int j) {
  const int off = j - i + d.es;
  if (off < 0 || off > d.es + d.er) return 0.0;
  return d.env[(size_t)i * (d.es + 1 + d.er) + off];
}

__device__ __forceinline__ void fail_dev(const LfDev& d, int errc, int detail) {
  if (threadIdx.x == 0) {
    d.st[ST_CODE] = 1 + errc;
    d.st[ST_DETAIL] = detail;
  }
}

// ---------------------------------------------------------------------------
// banded core (Lu / Lud): src/localfact.cpp:84-225
// ---------------------------------------------------------------------------

// x <- N^{-1} x on one column (stride = row pitch of the column's matrix)
__device__ void banded_n_inv(const LfDev& d, double* x, int stride) {
  const int L = d.L, es = d.es, er = d.er, w = es + 1 + er;
  for (int i = 0; i < L; ++i) {  // unit lower L
    double acc = x[(size_t)i * stride];
    const int dl = min(es, i);
    for (int q = 1; q <= dl; ++q) acc -= d.fac[(size_t)i * w + (es - q)] * x[(size_t)(i - q) * stride];
    x[(size_t)i * stride] = acc;
  }
  if (d.strategy != PSG_LUD) return;
  for (int i = L - 1; i >= 0; --i) {  // unit upper U' = U D^{-1}
    double acc = x[(size_t)i * stride];
    const int dl = min(er, L - 1 - i);
    for (int q = 1; q <= dl; ++q)
      acc -= (d.fac[(size_t)i * w + (es + q)] / d.dvec[i + q]) * x[(size_t)(i + q) * stride];
    x[(size_t)i * stride] = acc;
  }
}

// x <- S^{-1} x (Lu: upper U; Lud: D)
__device__ void banded_s_inv(const LfDev& d, double* x, int stride) {
  const int L = d.L, es = d.es, er = d.er, w = es + 1 + er;
  if (d.strategy == PSG_LUD) {
    for (int i = 0; i < L; ++i) x[(size_t)i * stride] /= d.dvec[i];
    return;
  }
  for (int i = L - 1; i >= 0; --i) {
    double acc = x[(size_t)i * stride];
    const int dl = min(er, L - 1 - i);
    for (int q = 1; q <= dl; ++q) acc -= d.fac[(size_t)i * w + (es + q)] * x[(size_t)(i + q) * stride];
    x[(size_t)i * stride] = acc / d.fac[(size_t)i * w + es];
  }
}

// x <- S^{-T} x
__device__ void banded_st_inv(const LfDev& d, double* x, int stride) {
  const int L = d.L, es = d.es, er = d.er, w = es + 1 + er;
  if (d.strategy == PSG_LUD) {
    for (int i = 0; i < L; ++i) x[(size_t)i * stride] /= d.dvec[i];
    return;
  }
  for (int i = 0; i < L; ++i) {
    double acc = x[(size_t)i * stride];
    const int dl = min(er, i);
    for (int q = 1; q <= dl; ++q) acc -= d.fac[(size_t)(i - q) * w + (es + q)] * x[(size_t)(i - q) * stride];
    x[(size_t)i * stride] = acc / d.fac[(size_t)i * w + es];
  }
}

// C(i,j) = sum_x A(x,i) B(x,j), x ascending, zero A entries skipped (at_b)
__device__ double at_b_entry(const double* A, int ka, const double* B, int kb, int L, int i, int j) {
  double acc = 0.0;
  for (int x = 0; x < L; ++x) {
    const double a = A[(size_t)x * ka + i];
    if (a == 0.0) continue;
    acc += a * B[(size_t)x * kb + j];
  }
  return acc;
}

// interface blocks and the kept block from the fill-ins (banded and dense
// cores share the layout of kept: [left | extras | right])
__device__ void banded_interface(const LfDev& d) {
  const int k0 = d.k0, k1 = d.k1, L = d.L, kd = k0 + k1;
  for (int e = threadIdx.x; e < k0 * k0; e += blockDim.x)
    d.a1[e] = -at_b_entry(d.w, k0, d.z, k0, L, e / k0, e % k0);
  for (int e = threadIdx.x; e < k1 * k1; e += blockDim.x)
    d.a2[e] = d.ar[e] - at_b_entry(d.v, k1, d.y, k1, L, e / k1, e % k1);
  for (int e = threadIdx.x; e < k1 * k0; e += blockDim.x)
    d.be[e] = -at_b_entry(d.v, k1, d.z, k0, L, e / k0, e % k0);
  for (int e = threadIdx.x; e < k0 * k1; e += blockDim.x)
    d.ga[e] = -at_b_entry(d.w, k0, d.y, k1, L, e / k1, e % k1);
  __syncthreads();
  for (int e = threadIdx.x; e < kd * kd; e += blockDim.x) {
    const int i = e / kd, j = e % kd;
    double val;
    if (i < k0)
      val = j < k0 ? d.a1[i * k0 + j] : d.ga[i * k1 + (j - k0)];
    else
      val = j < k0 ? d.be[(i - k0) * k0 + j] : d.a2[(i - k0) * k1 + (j - k0)];
    d.kept[e] = val;
  }
}

__global__ void __launch_bounds__(kThreads) lf_banded_kernel(LfDev d) {
  const int L = d.L, es = d.es, er = d.er, w = es + 1 + er, tid = threadIdx.x, nt = blockDim.x;
  for (size_t e = tid; e < (size_t)L * w; e += nt) d.fac[e] = d.env[e];
  __syncthreads();
  // no-pivot band elimination, pivot by pivot (banded_eliminate, :84-100)
  for (int k = 0; k < L; ++k) {
    const double dk = d.fac[(size_t)k * w + es];
    if (dk == 0.0) {
      fail_dev(d, PSG_E_ZERO_PIVOT, k);
      return;
    }
    const int ni = min(L - 1, k + es) - k, nj = min(L - 1, k + er) - k;
    for (int t = tid; t < ni; t += nt) {
      const double e = d.fac[(size_t)(k + 1 + t) * w + (es - 1 - t)];
      d.flag[t] = e != 0.0;
      d.mu[t] = e / dk;
    }
    __syncthreads();
    for (int idx = tid; idx < ni * nj; idx += nt) {
      const int t = idx / nj, u = idx % nj;
      if (!d.flag[t]) continue;
      const int i = k + 1 + t, j = k + 1 + u;
      double& e = d.fac[(size_t)i * w + (j - i + es)];
      e = e - d.mu[t] * d.fac[(size_t)k * w + (j - k + es)];
    }
    for (int t = tid; t < ni; t += nt)
      if (d.flag[t]) d.fac[(size_t)(k + 1 + t) * w + (es - 1 - t)] = d.mu[t];
    __syncthreads();
  }
  if (d.strategy == PSG_LUD)
    for (int i = tid; i < L; i += nt) d.dvec[i] = d.fac[(size_t)i * w + es];
  __syncthreads();
  // fill-ins z = N^-1 b0, y = N^-1 c1, w = S^-T c0, v = S^-T b1 (:202-205), one column per thread
  const int k0 = d.k0, k1 = d.k1;
  for (int c = tid; c < 2 * (k0 + k1); c += nt) {
    const double* src;
    double* dst;
    int kk, col;
    bool n_side;
    if (c < k0) { src = d.b0; dst = d.z; kk = k0; col = c; n_side = true; }
    else if (c < k0 + k1) { src = d.c1; dst = d.y; kk = k1; col = c - k0; n_side = true; }
    else if (c < 2 * k0 + k1) { src = d.c0; dst = d.w; kk = k0; col = c - k0 - k1; n_side = false; }
    else { src = d.b1; dst = d.v; kk = k1; col = c - 2 * k0 - k1; n_side = false; }
    for (int i = 0; i < L; ++i) dst[(size_t)i * kk + col] = src[(size_t)i * kk + col];
    if (n_side) banded_n_inv(d, dst + col, kk);
    else banded_st_inv(d, dst + col, kk);
  }
  __syncthreads();
  banded_interface(d);
}

// ---------------------------------------------------------------------------
// cyclic reduction core: src/localfact.cpp:266-384
// ---------------------------------------------------------------------------

// C = A (ra x ca) * B (ca x cb), entry-parallel, k ascending, zero A skipped (matmul)
__device__ void cta_mm(const double* A, const double* B, double* C, int ra, int ca, int cb) {
  for (int e = threadIdx.x; e < ra * cb; e += blockDim.x) {
    const int i = e / cb, j = e % cb;
    double acc = 0.0;
    for (int k = 0; k < ca; ++k) {
      const double a = A[i * ca + k];
      if (a == 0.0) continue;
      acc += a * B[k * cb + j];
    }
    C[e] = acc;
  }
  __syncthreads();
}

// Ainv = inverse(A), n x n: LU with partial pivoting on one thread, then one
// identity column per thread (DenseLu + DenseLu::solve).  false if singular.
__device__ bool cta_inverse(const LfDev& d, const double* A, double* Ainv, int n) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    double* lu = d.lu;
    int* perm = d.perm;
    for (int e = 0; e < n * n; ++e) lu[e] = A[e];
    for (int i = 0; i < n; ++i) perm[i] = i;
    int ok = 1;
    for (int k = 0; k < n && ok; ++k) {
      int piv = k;
      double best = fabs(lu[k * n + k]);
      for (int i = k + 1; i < n; ++i) {
        const double v = fabs(lu[i * n + k]);
        if (v > best) { best = v; piv = i; }
      }
      if (best == 0.0) { ok = 0; break; }
      if (piv != k) {
        for (int j = 0; j < n; ++j) {
          const double t = lu[k * n + j];
          lu[k * n + j] = lu[piv * n + j];
          lu[piv * n + j] = t;
        }
        const int t = perm[k];
        perm[k] = perm[piv];
        perm[piv] = t;
      }
      const double dk = lu[k * n + k];
      for (int i = k + 1; i < n; ++i) {
        const double m = lu[i * n + k] / dk;
        lu[i * n + k] = m;
        if (m == 0.0) continue;
        for (int j = k + 1; j < n; ++j) lu[i * n + j] -= m * lu[k * n + j];
      }
    }
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return false;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double* lu = d.lu;
    double* y = Ainv + j;  // column j, stride n
    for (int i = 0; i < n; ++i) y[i * n] = d.perm[i] == j ? 1.0 : 0.0;
    for (int i = 0; i < n; ++i)
      for (int q = 0; q < i; ++q) y[i * n] -= lu[i * n + q] * y[q * n];
    for (int i = n - 1; i >= 0; --i) {
      for (int q = i + 1; q < n; ++q) y[i * n] -= lu[i * n + q] * y[q * n];
      y[i * n] /= lu[i * n + i];
    }
  }
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(kThreads) lf_cr_kernel(LfDev d) {
  const int g = d.g, gg = g * g, nb = d.nb, tid = threadIdx.x, nt = blockDim.x;
  const int k0 = d.k0, k1 = d.k1, kd = k0 + k1, L = d.L;
  double *A = d.ca, *D = d.cd, *C = d.cc;
  for (int e = tid; e < nb * gg; e += nt) {
    const int j = e / gg, ti = (e % gg) / g, tj = e % g;
    D[e] = body_at(d, j * g + ti, j * g + tj);
    A[e] = j > 0 ? body_at(d, j * g + ti, (j - 1) * g + tj) : 0.0;
    C[e] = j < nb - 1 ? body_at(d, j * g + ti, (j + 1) * g + tj) : 0.0;
  }
  for (int j = tid; j < nb; j += nt) d.act[j] = j;
  __syncthreads();
  int nact = nb, levels = 0, nel = 0;
  while (nact > 2) {
    ++levels;
    int nkeep = 1;
    if (tid == 0) d.keep[0] = d.act[0];
    __syncthreads();
    int idx = 1;
    while (idx + 1 < nact) {
      const int j = d.act[idx], l = d.keep[nkeep - 1], rn = d.act[idx + 1];
      int* ei = d.elim_idx + 3 * nel;
      double* em = d.elim_mat + (size_t)nel * 5 * gg;
      double *ml = em, *mr = em + gg, *ea = em + 2 * gg, *ec = em + 3 * gg, *dinv = em + 4 * gg;
      if (tid == 0) { ei[0] = j; ei[1] = l; ei[2] = rn; }
      if (!cta_inverse(d, D + (size_t)j * gg, dinv, g)) {
        fail_dev(d, PSG_E_ZERO_PIVOT, j * g);
        return;
      }
      for (int e = tid; e < gg; e += nt) {
        ea[e] = A[(size_t)j * gg + e];
        ec[e] = C[(size_t)j * gg + e];
      }
      __syncthreads();
      cta_mm(C + (size_t)l * gg, dinv, ml, g, g, g);   // ml = c[l] dinv
      cta_mm(A + (size_t)rn * gg, dinv, mr, g, g, g);  // mr = a[rn] dinv
      cta_mm(ml, ea, d.tmp, g, g, g);
      for (int e = tid; e < gg; e += nt) D[(size_t)l * gg + e] -= d.tmp[e];  // d[l] -= ml a
      __syncthreads();
      cta_mm(ml, ec, d.tmp, g, g, g);
      for (int e = tid; e < gg; e += nt) C[(size_t)l * gg + e] = -d.tmp[e];  // c[l] = -ml c
      __syncthreads();
      cta_mm(mr, ec, d.tmp, g, g, g);
      for (int e = tid; e < gg; e += nt) D[(size_t)rn * gg + e] -= d.tmp[e];  // d[rn] -= mr c
      __syncthreads();
      cta_mm(mr, ea, d.tmp, g, g, g);
      for (int e = tid; e < gg; e += nt) A[(size_t)rn * gg + e] = -d.tmp[e];  // a[rn] = -mr a
      if (tid == 0) d.keep[nkeep] = rn;
      __syncthreads();
      ++nkeep;
      ++nel;
      idx += 2;
    }
    if (d.keep[nkeep - 1] != d.act[nact - 1]) {
      if (tid == 0) d.keep[nkeep] = d.act[nact - 1];
      ++nkeep;
    }
    __syncthreads();
    for (int q = tid; q < nkeep; q += nt) d.act[q] = d.keep[q];
    nact = nkeep;
    __syncthreads();
  }
  const int R = nact, rg = R * g;
  // remaining system d2 and its inverse
  for (int e = tid; e < rg * rg; e += nt) {
    const int i = e / rg, j = e % rg, u = i / g, q = j / g, ti = i % g, tj = j % g;
    double val = 0.0;
    if (u == q) val = D[(size_t)d.act[u] * gg + ti * g + tj];
    else if (u == 0) val = C[(size_t)d.act[0] * gg + ti * g + tj];
    else val = A[(size_t)d.act[1] * gg + ti * g + tj];
    d.d2[e] = val;
  }
  __syncthreads();
  if (!cta_inverse(d, d.d2, d.d2inv, rg)) {
    fail_dev(d, PSG_E_ZERO_PIVOT, d.act[0] * g);
    return;
  }
  // couplings of the remaining rows to the separators (no fill-in vectors)
  for (int e = tid; e < rg * kd; e += nt) {
    const int q = e / kd, c = e % kd;
    double val = 0.0;
    if (c < k0) { if (q < g && q < L) val = d.b0[(size_t)q * k0 + c]; }
    if (c >= k0 && q >= rg - g) {
      const int ti = q - (rg - g);
      if (ti < L) val = d.c1[(size_t)(L - g + ti) * k1 + (c - k0)];
    }
    d.cmat[e] = val;
  }
  for (int e = tid; e < kd * rg; e += nt) {
    const int i = e / rg, q = e % rg;
    double val = 0.0;
    if (i < k0) { if (q < g && q < L) val = d.c0[(size_t)q * k0 + i]; }
    else if (q >= rg - g) {
      const int ti = q - (rg - g);
      if (ti < L) val = d.b1[(size_t)(L - g + ti) * k1 + (i - k0)];
    }
    d.rmat[e] = val;
  }
  __syncthreads();
  cta_mm(d.rmat, d.d2inv, d.rmd2, kd, rg, rg);
  cta_mm(d.rmd2, d.cmat, d.corr, kd, rg, kd);
  for (int e = tid; e < kd * kd; e += nt) {
    const int i = e / kd, j = e % kd;
    double val = (i >= k0 && j >= k0) ? d.ar[(i - k0) * k1 + (j - k0)] : 0.0;
    val -= d.corr[e];
    d.kept[e] = val;
  }
  __syncthreads();
  for (int e = tid; e < kd * kd; e += nt) {
    const int i = e / kd, j = e % kd;
    const double val = d.kept[e];
    if (i < k0) {
      if (j < k0) d.a1[i * k0 + j] = val; else d.ga[i * k1 + (j - k0)] = val;
    } else {
      if (j < k0) d.be[(i - k0) * k0 + j] = val; else d.a2[(i - k0) * k1 + (j - k0)] = val;
    }
  }
  if (tid == 0) {
    d.st[ST_NELIM] = nel;
    d.st[ST_LEVELS] = levels;
    d.st[ST_NREM] = R;
    d.st[ST_REM0] = d.act[0];
    d.st[ST_REM1] = R > 1 ? d.act[1] : -1;
  }
}

// ---------------------------------------------------------------------------
// dense recorded core (LuPivot / Qr): src/localfact.cpp:400-700
// ---------------------------------------------------------------------------

// rows rho in [lo, hi) with rowsel(rho): CTA argmax of |W(rho, col)|, ties to
// the lowest row, NaN never wins (the serial scan with best = -1, strict >)
template <typename Sel>
__device__ void cta_argmax(const double* W, int dim, int col, int lo, int hi, Sel rowsel, double* best_out,
                           int* idx_out) {
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  double best = -1.0;
  int bi = -1;
  for (int rho = lo + threadIdx.x; rho < hi; rho += blockDim.x) {
    if (!rowsel(rho)) continue;
    const double v = fabs(W[(size_t)rho * dim + col]);
    if (v > best) { best = v; bi = rho; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, best, o);
    const int oi = __shfl_down_sync(0xffffffffu, bi, o);
    if (oi >= 0 && (ov > best || (ov == best && (bi < 0 || oi < bi)))) { best = ov; bi = oi; }
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) { s_v[wid] = best; s_i[wid] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = -1.0;
    int i = -1;
    for (int q = 0; q < nw; ++q)
      if (s_i[q] >= 0 && (s_v[q] > b || (s_v[q] == b && (i < 0 || s_i[q] < i)))) { b = s_v[q]; i = s_i[q]; }
    s_v[0] = b;
    s_i[0] = i;
  }
  __syncthreads();
  *best_out = s_v[0];
  *idx_out = s_i[0];
  __syncthreads();
}

// rowop(rho, piv, mu) for every selected row rho (ascending), the way
// eliminate_column issues them: mu from W(rho, col) / W(piv, col); W and
// Lmat rows are independent, Linv(:, piv) accumulates in rho order.
template <typename Sel>
__device__ void cta_eliminate(const LfDev& d, int col, int piv, Sel rowsel) {
  const int dim = d.dim, tid = threadIdx.x, nt = blockDim.x;
  double* W = d.W;
  const double wp = W[(size_t)piv * dim + col];
  for (int rho = tid; rho < dim; rho += nt) {
    int f = 0;
    if (rho != piv && rowsel(rho)) {
      const double e = W[(size_t)rho * dim + col];
      if (e != 0.0) {
        const double mu = e / wp;
        d.vv[rho] = mu;
        f = mu != 0.0 ? 2 : 1;  // 1: entry cleared, rowop a no-op (mu underflowed)
      }
    }
    d.row_state[dim + rho] = f;  // scratch flags behind row_state
  }
  __syncthreads();
  const int* flag = d.row_state + dim;
  for (size_t e = tid; e < (size_t)dim * dim; e += nt) {
    const int rho = int(e / dim), j = int(e % dim);
    if (flag[rho] != 2) continue;
    const double mu = d.vv[rho];
    W[e] -= mu * W[(size_t)piv * dim + j];
    d.Lm[e] -= mu * d.Lm[(size_t)piv * dim + j];
  }
  for (int i = tid; i < dim; i += nt) {
    double acc = d.Li[(size_t)i * dim + piv];
    for (int rho = 0; rho < dim; ++rho)
      if (flag[rho] == 2) acc += d.vv[rho] * d.Li[(size_t)i * dim + rho];
    d.Li[(size_t)i * dim + piv] = acc;
  }
  __syncthreads();
  for (int rho = tid; rho < dim; rho += nt)
    if (flag[rho]) W[(size_t)rho * dim + col] = 0.0;
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) lf_dense_kernel(LfDev d) {
  const int dim = d.dim, k0 = d.k0, k1 = d.k1, L = d.L, tid = threadIdx.x, nt = blockDim.x;
  double *W = d.W, *Lm = d.Lm, *Li = d.Li;
  // frame = local_dense(blk), Lmat = Linv = I
  for (size_t e = tid; e < (size_t)dim * dim; e += nt) {
    const int i = int(e / dim), j = int(e % dim);
    double val = 0.0;
    const bool bi = i >= k0 && i < k0 + L, bj = j >= k0 && j < k0 + L;
    if (bi && bj) val = body_at(d, i - k0, j - k0);
    else if (bi && j < k0) val = d.b0[(size_t)(i - k0) * k0 + j];
    else if (bj && i < k0) val = d.c0[(size_t)(j - k0) * k0 + i];
    else if (bi && j >= k0 + L) val = d.c1[(size_t)(i - k0) * k1 + (j - k0 - L)];
    else if (bj && i >= k0 + L) val = d.b1[(size_t)(j - k0) * k1 + (i - k0 - L)];
    else if (i >= k0 + L && j >= k0 + L) val = d.ar[(i - k0 - L) * k1 + (j - k0 - L)];
    W[e] = val;
    Lm[e] = Li[e] = i == j ? 1.0 : 0.0;
  }
  for (int i = tid; i < dim; i += nt) {
    const bool sep = i < k0 || i >= k0 + L;
    d.row_state[i] = sep ? 3 : 0;
    d.col_state[i] = sep ? 2 : 0;
  }
  __shared__ double s_scale;
  if (tid == 0) {  // body_scale: largest absolute envelope row sum
    double best = 1e-300;
    const int w = d.es + 1 + d.er;
    for (int i = 0; i < L; ++i) {
      double s = 0.0;
      for (int q = 0; q < w; ++q) s += fabs(d.env[(size_t)i * w + q]);
      best = fmax(best, s);
    }
    s_scale = best;
  }
  __syncthreads();
  const double thresh = d.tol * s_scale;
  int naord = 0, ndef = 0;
  int* rs = d.row_state;
  if (d.strategy == PSG_LUPIVOT) {
    for (int t = 0; t < L; ++t) {
      const int col = k0 + t;
      double best;
      int piv;
      cta_argmax(W, dim, col, k0, k0 + L, [&](int rho) { return rs[rho] == 0; }, &best, &piv);
      if (best < thresh) {  // deferred: the lowest active row joins the reduced system
        if (tid == 0) {
          int rho = -1;
          for (int q = k0; q < k0 + L; ++q)
            if (rs[q] == 0) { rho = q; break; }
          rs[rho] = 4;
          d.col_state[col] = 3;
          d.deferred[2 * ndef] = rho;
          d.deferred[2 * ndef + 1] = col;
        }
        ++ndef;
        __syncthreads();
        continue;
      }
      if (tid == 0) {
        rs[piv] = 1;
        d.col_state[col] = 1;
        d.a_order[2 * naord] = piv;
        d.a_order[2 * naord + 1] = col;
      }
      ++naord;
      __syncthreads();
      cta_eliminate(d, col, piv, [&](int rho) { return rs[rho] != 1 && rs[rho] != 2; });
    }
  } else {  // Qr: Householder reflectors over the active rows act = [k0 + h, k0 + L)
    __shared__ double s_nrm, s_tau, s_alpha;
    int h = 0;
    for (int t = 0; t < L; ++t) {
      const int col = k0 + t, lo = k0 + h, na = L - h;
      if (tid == 0) {
        double nrm2 = 0.0;
        for (int u = 0; u < na; ++u) {
          const double x = W[(size_t)(lo + u) * dim + col];
          nrm2 += x * x;
        }
        s_nrm = sqrt(nrm2);
      }
      __syncthreads();
      const double nrm = s_nrm;
      if (nrm < thresh) {
        if (tid == 0) {
          rs[lo] = 4;
          d.col_state[col] = 3;
          d.deferred[2 * ndef] = lo;
          d.deferred[2 * ndef + 1] = col;
        }
        ++ndef;
        ++h;
        __syncthreads();
        continue;
      }
      if (tid == 0) {
        const double x0 = W[(size_t)lo * dim + col];
        const double alpha = x0 >= 0 ? -nrm : nrm;
        double vtv = 0.0;
        for (int u = 0; u < na; ++u) {
          double q = W[(size_t)(lo + u) * dim + col];
          if (u == 0) q -= alpha;
          d.vv[u] = q;
          vtv += q * q;
        }
        s_alpha = alpha;
        s_tau = vtv > 0.0 ? 2.0 / vtv : 0.0;
      }
      __syncthreads();
      if (s_tau != 0.0) {  // reflect(act, v, tau) on W, Lmat (columns) and Linv (rows)
        const double tau = s_tau;
        for (int j = tid; j < 2 * dim; j += nt) {
          double* M = j < dim ? W : Lm;
          const int jj = j < dim ? j : j - dim;
          double s = 0.0;
          for (int u = 0; u < na; ++u) s += d.vv[u] * M[(size_t)(lo + u) * dim + jj];
          s *= tau;
          for (int u = 0; u < na; ++u) M[(size_t)(lo + u) * dim + jj] -= s * d.vv[u];
        }
        for (int i = tid; i < dim; i += nt) {
          double s = 0.0;
          for (int u = 0; u < na; ++u) s += d.vv[u] * Li[(size_t)i * dim + lo + u];
          s *= tau;
          for (int u = 0; u < na; ++u) Li[(size_t)i * dim + lo + u] -= s * d.vv[u];
        }
        __syncthreads();
      }
      for (int u = tid; u < na; u += nt) W[(size_t)(lo + u) * dim + col] = u == 0 ? s_alpha : 0.0;
      if (tid == 0) {
        rs[lo] = 1;
        d.col_state[col] = 1;
        d.a_order[2 * naord] = lo;
        d.a_order[2 * naord + 1] = col;
      }
      ++naord;
      ++h;
      __syncthreads();
    }
    // separator and deferred rows condensed against the R rows
    for (int q = 0; q < naord; ++q) {
      const int piv = d.a_order[2 * q], col = d.a_order[2 * q + 1];
      cta_eliminate(d, col, piv, [&](int rho) { return rs[rho] == 3 || rs[rho] == 4; });
    }
  }
  if (ndef == L) {
    fail_dev(d, PSG_E_EXHAUSTED_BODY, 0);
    return;
  }
  // finish_dense + dense_factor: kept rows/cols, pivot pairing, interface views
  const int kd = k0 + ndef + k1;
  for (int u = tid; u < kd; u += nt) {
    int rr, cc;
    if (u < k0) rr = cc = u;
    else if (u < k0 + ndef) { rr = d.deferred[2 * (u - k0)]; cc = d.deferred[2 * (u - k0) + 1]; }
    else rr = cc = k0 + L + (u - k0 - ndef);
    d.kept_rows[u] = rr;
    d.kept_cols[u] = cc;
  }
  for (int j = tid; j < dim; j += nt) d.pair_row[j] = j;
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < naord; ++q) d.pair_row[d.a_order[2 * q + 1]] = d.a_order[2 * q];
    for (int u = 0; u < kd; ++u) d.pair_row[d.kept_cols[u]] = d.kept_rows[u];
  }
  __syncthreads();
  for (int u = tid; u < ndef; u += nt) {
    d.ext_pos[u] = d.kept_cols[k0 + u] - k0;
    d.ext_alpha[u] = W[(size_t)d.kept_rows[k0 + u] * dim + d.kept_cols[k0 + u]];
  }
  for (int x = tid; x < L; x += nt) {
    const int rho = d.pair_row[k0 + x];
    bool kept_col = false;
    for (int u = 0; u < kd; ++u)
      if (d.kept_cols[u] == k0 + x) kept_col = true;
    for (int t = 0; t < k0; ++t) {
      d.w[(size_t)x * k0 + t] = Li[(size_t)t * dim + rho];
      d.z[(size_t)x * k0 + t] = kept_col ? 0.0 : W[(size_t)rho * dim + t];
    }
    for (int t = 0; t < k1; ++t) {
      d.v[(size_t)x * k1 + t] = Li[(size_t)(k0 + L + t) * dim + rho];
      d.y[(size_t)x * k1 + t] = kept_col ? 0.0 : W[(size_t)rho * dim + k0 + L + t];
    }
  }
  for (int e = tid; e < k0 * k0; e += nt) d.a1[e] = W[(size_t)(e / k0) * dim + e % k0];
  for (int e = tid; e < k0 * k1; e += nt) d.ga[e] = W[(size_t)(e / k1) * dim + k0 + L + e % k1];
  for (int e = tid; e < k1 * k0; e += nt) d.be[e] = W[(size_t)(k0 + L + e / k0) * dim + e % k0];
  for (int e = tid; e < k1 * k1; e += nt) d.a2[e] = W[(size_t)(k0 + L + e / k1) * dim + k0 + L + e % k1];
  for (int e = tid; e < kd * kd; e += nt)
    d.kept[e] = W[(size_t)d.kept_rows[e / kd] * dim + d.kept_cols[e % kd]];
  if (tid == 0) {
    d.st[ST_NAORD] = naord;
    d.st[ST_NDEF] = ndef;
  }
}

// ---------------------------------------------------------------------------
// member operations: condense / backsolve / apply_N_inv / apply_S_inv
// (src/localfact.cpp:765-875).  io: [0, L) body vector, [L, L+kd) kept vector,
// [L+kd, L+kd+L) second body vector, scratch behind.
// ---------------------------------------------------------------------------
enum { OP_CONDENSE = 0, OP_BACKSOLVE = 1, OP_NINV = 2, OP_SINV = 3 };

__device__ void cr_forward(const LfDev& d, int nel, double* t) {  // block_axpy sequence
  const int g = d.g, gg = g * g;
  for (int q = 0; q < nel; ++q) {
    const int* ei = d.elim_idx + 3 * q;
    const double* em = d.elim_mat + (size_t)q * 5 * gg;
    for (int side = 0; side < 2; ++side) {
      const double* M = em + side * gg;
      const int tgt = ei[1 + side], src = ei[0];
      for (int ti = 0; ti < g; ++ti) {
        double acc = 0.0;
        for (int tj = 0; tj < g; ++tj) acc += M[ti * g + tj] * t[(size_t)src * g + tj];
        t[(size_t)tgt * g + ti] -= acc;
      }
    }
  }
}

// frame matvec t = Lmat [0; body; 0] (row-parallel)
__device__ void dense_lmat_apply(const LfDev& d, const double* body, double* t) {
  const int dim = d.dim, k0 = d.k0, L = d.L;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < dim; ++j) {
      const double fj = (j >= k0 && j < k0 + L) ? body[j - k0] : 0.0;
      s += d.Lm[(size_t)i * dim + j] * fj;
    }
    t[i] = s;
  }
  __syncthreads();
}

__device__ void backsolve_dev(const LfDev& d, int kd, int naord, int nel, int nrem, const int* rem,
                              const double* ghat, const double* xk, double* x, double* scr) {
  const int L = d.L, k0 = d.k0, k1 = d.k1, tid = threadIdx.x;
  if (d.strategy == PSG_LU || d.strategy == PSG_LUD) {
    for (int i = tid; i < L; i += blockDim.x) {
      double acc = ghat[i];
      for (int t = 0; t < k0; ++t) acc -= d.z[(size_t)i * k0 + t] * xk[t];
      for (int t = 0; t < k1; ++t) acc -= d.y[(size_t)i * k1 + t] * xk[k0 + t];
      x[i] = acc;
    }
    __syncthreads();
    if (tid == 0) banded_s_inv(d, x, 1);
    return;
  }
  if (d.strategy == PSG_CR) {
    if (tid != 0) return;
    const int g = d.g, gg = g * g, rg = nrem * g;
    double* trem = scr;
    double* xrem = scr + rg;
    for (int u = 0; u < nrem; ++u)
      for (int t = 0; t < g; ++t) trem[u * g + t] = ghat[(size_t)rem[u] * g + t];
    for (int q = 0; q < rg; ++q)
      for (int i = 0; i < kd; ++i) trem[q] -= d.cmat[q * kd + i] * xk[i];
    for (int q = 0; q < rg; ++q) {
      double s = 0.0;
      for (int j = 0; j < rg; ++j) s += d.d2inv[q * rg + j] * trem[j];
      xrem[q] = s;
    }
    for (int i = 0; i < L; ++i) x[i] = 0.0;
    for (int u = 0; u < nrem; ++u)
      for (int t = 0; t < g; ++t) x[(size_t)rem[u] * g + t] = xrem[u * g + t];
    double* rhs = xrem + rg;
    for (int q = nel - 1; q >= 0; --q) {
      const int* ei = d.elim_idx + 3 * q;
      const double* em = d.elim_mat + (size_t)q * 5 * gg;
      const double *ea = em + 2 * gg, *ec = em + 3 * gg, *dinv = em + 4 * gg;
      for (int t = 0; t < g; ++t) rhs[t] = ghat[(size_t)ei[0] * g + t];
      for (int t = 0; t < g; ++t) {
        double acc = rhs[t];
        for (int u = 0; u < g; ++u) acc -= ea[t * g + u] * x[(size_t)ei[1] * g + u];
        for (int u = 0; u < g; ++u) acc -= ec[t * g + u] * x[(size_t)ei[2] * g + u];
        rhs[t] = acc;
      }
      for (int t = 0; t < g; ++t) {
        double acc = 0.0;
        for (int u = 0; u < g; ++u) acc += dinv[t * g + u] * rhs[u];
        x[(size_t)ei[0] * g + t] = acc;
      }
    }
    return;
  }
  // dense recorded core: substitution in reverse pivot order
  if (tid != 0) return;
  const int dim = d.dim;
  double* xi = scr;
  for (int j = 0; j < dim; ++j) xi[j] = 0.0;
  for (int i = 0; i < kd; ++i) xi[d.kept_cols[i]] = xk[i];
  for (int q = naord - 1; q >= 0; --q) {
    const int rho = d.a_order[2 * q], c = d.a_order[2 * q + 1];
    double acc = (rho >= k0 && rho < k0 + L) ? ghat[rho - k0] : 0.0;
    for (int j = 0; j < dim; ++j) {
      if (j == c) continue;
      const double e = d.W[(size_t)rho * dim + j];
      if (e != 0.0) acc -= e * xi[j];
    }
    xi[c] = acc / d.W[(size_t)rho * dim + c];
  }
  for (int x_ = 0; x_ < L; ++x_) x[x_] = xi[k0 + x_];
}

__global__ void __launch_bounds__(kThreads) lf_op_kernel(LfDev d, int op, double* io, double* scr) {
  const int L = d.L, k0 = d.k0, k1 = d.k1, tid = threadIdx.x;
  const int naord = d.st[ST_NAORD], ndef = d.st[ST_NDEF], nel = d.st[ST_NELIM], nrem = d.st[ST_NREM];
  const int rem[2] = {d.st[ST_REM0], d.st[ST_REM1]};
  const int kd = k0 + k1 + (d.strategy == PSG_LUPIVOT || d.strategy == PSG_QR ? ndef : 0);
  double *vb = io, *vk = io + L, *vo = io + L + kd;
  const bool banded = d.strategy == PSG_LU || d.strategy == PSG_LUD;
  if (op == OP_CONDENSE || op == OP_NINV) {  // body vector vb -> ghat (vo); condense also kept_rhs (vk)
    if (banded) {
      if (tid == 0) {
        for (int i = 0; i < L; ++i) vo[i] = vb[i];
        banded_n_inv(d, vo, 1);
      }
      __syncthreads();
      if (op == OP_CONDENSE)
        for (int t = tid; t < kd; t += blockDim.x) {
          const double* M = t < k0 ? d.w : d.v;
          const int kk = t < k0 ? k0 : k1, c = t < k0 ? t : t - k0;
          double acc = 0.0;
          for (int x = 0; x < L; ++x) acc += M[(size_t)x * kk + c] * vo[x];
          vk[t] = -acc;
        }
    } else if (d.strategy == PSG_CR) {
      if (tid == 0) {
        for (int i = 0; i < L; ++i) vo[i] = vb[i];
        cr_forward(d, nel, vo);
      }
      __syncthreads();
      if (op == OP_CONDENSE) {
        const int g = d.g, rg = nrem * g;
        for (int i = tid; i < kd; i += blockDim.x) {
          double acc = 0.0;
          for (int q = 0; q < rg; ++q) acc += d.rmd2[i * rg + q] * vo[(size_t)rem[q / g] * g + q % g];
          vk[i] = -acc;
        }
      }
    } else {
      dense_lmat_apply(d, vb, scr);
      for (int x = tid; x < L; x += blockDim.x) vo[x] = op == OP_CONDENSE ? scr[k0 + x] : scr[d.pair_row[k0 + x]];
      if (op == OP_CONDENSE)
        for (int i = tid; i < kd; i += blockDim.x) vk[i] = scr[d.kept_rows[i]];
    }
    return;
  }
  if (op == OP_SINV && banded) {
    if (tid == 0) {
      for (int i = 0; i < L; ++i) vo[i] = vb[i];
      banded_s_inv(d, vo, 1);
    }
    return;
  }
  if (op == OP_SINV)  // backsolve with zero kept values
    for (int i = tid; i < kd; i += blockDim.x) vk[i] = 0.0;
  __syncthreads();
  backsolve_dev(d, kd, naord, nel, nrem, rem, vb, vk, vo, scr);
}

// ---------------------------------------------------------------------------
// dense reduced solve (solve_reduced on an explicit T): LU with partial
// pivoting, one launch pair per column, bit-identical to src/parfact.cpp:134-184
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) ds_pivot_kernel(double* lu, int* perm, int n, int c, int* bad) {
  if (*bad) return;
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  __shared__ int s_piv;
  double best = -1.0;
  int bi = -1;
  for (int i = c + 1 + threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(lu[(size_t)i * n + c]);
    if (v > best) { best = v; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, best, o);
    const int oi = __shfl_down_sync(0xffffffffu, bi, o);
    if (oi >= 0 && (ov > best || (ov == best && (bi < 0 || oi < bi)))) { best = ov; bi = oi; }
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) { s_v[wid] = best; s_i[wid] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = fabs(lu[(size_t)c * n + c]);  // the serial scan starts at the diagonal
    int piv = c;
    double rb = -1.0;
    int ri = -1;
    for (int q = 0; q < nw; ++q)
      if (s_i[q] >= 0 && (s_v[q] > rb || (s_v[q] == rb && (ri < 0 || s_i[q] < ri)))) { rb = s_v[q]; ri = s_i[q]; }
    if (ri >= 0 && rb > b) { b = rb; piv = ri; }
    if (b == 0.0) *bad = 1 + c;
    s_piv = piv;
  }
  __syncthreads();
  if (*bad) return;
  const int piv = s_piv;
  if (piv != c) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double t = lu[(size_t)c * n + j];
      lu[(size_t)c * n + j] = lu[(size_t)piv * n + j];
      lu[(size_t)piv * n + j] = t;
    }
    if (threadIdx.x == 0) {
      const int t = perm[c];
      perm[c] = perm[piv];
      perm[piv] = t;
    }
  }
  __syncthreads();
  const double dc = lu[(size_t)c * n + c];
  for (int i = c + 1 + threadIdx.x; i < n; i += blockDim.x) lu[(size_t)i * n + c] = lu[(size_t)i * n + c] / dc;
}

__global__ void ds_update_kernel(double* lu, int n, int c, const int* bad) {
  if (*bad) return;
  const int m = n - c - 1;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)m * m; e += (size_t)gridDim.x * blockDim.x) {
    const int i = c + 1 + int(e / m), j = c + 1 + int(e % m);
    lu[(size_t)i * n + j] -= lu[(size_t)i * n + c] * lu[(size_t)c * n + j];
  }
}

__global__ void ds_subst_kernel(const double* lu, const int* perm, int n, const double* rhs, double* x, const int* bad) {
  if (*bad || threadIdx.x != 0) return;
  for (int i = 0; i < n; ++i) x[i] = rhs[perm[i]];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= lu[(size_t)i * n + j] * x[j];
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) x[i] -= lu[(size_t)i * n + j] * x[j];
    x[i] /= lu[(size_t)i * n + i];
  }
}

__global__ void ds_iota_kernel(int* perm, int n, int* bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) perm[i] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) *bad = 0;
}

// arena of one local factorization
struct Arena {
  std::vector<size_t> off;
  size_t bytes = 0;
  size_t take(size_t count, size_t elem) {
    bytes = (bytes + 15) & ~size_t(15);
    const size_t o = bytes;
    bytes += std::max<size_t>(count, 1) * elem;
    return o;
  }
};

}  // namespace

struct psg_local {
  LfDev d{};
  char* base = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  int st[ST_COUNT] = {};
  size_t io_off = 0, scr_off = 0;
  int kd() const {
    return d.k0 + d.k1 + ((d.strategy == PSG_LUPIVOT || d.strategy == PSG_QR) ? st[ST_NDEF] : 0);
  }
  ~psg_local() {
    if (base) cudaFree(base);
  }
};

namespace {

struct DevGuard {
  int prev = -1, want;
  explicit DevGuard(int d) : want(d) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

const char* errc_text(int code) {
  switch (code) {
    case PSG_E_ZERO_PIVOT: return "zero pivot";
    case PSG_E_EXHAUSTED_BODY: return "exhausted body";
    default: return "error";
  }
}

}  // namespace

extern "C" {

int psg_local_factor(const psg_block* blk, int strategy, double tol, void* stream, psg_local** out, char* err,
                     size_t errlen) {
  if (!blk || !out) return lf_err(err, errlen, PSG_E_INVALID_PARAMETER, "null argument");
  *out = nullptr;
  const int L = blk->L, k0 = blk->k0, k1 = blk->k1, es = blk->env_s, er = blk->env_r;
  if (L < 1 || k0 < 0 || k1 < 0 || es < 0 || er < 0 || (L > 0 && (es > L - 1 || er > L - 1)))
    return lf_err(err, errlen, PSG_E_DIMENSION_MISMATCH, "block shape");
  if (strategy == PSG_ARCE)
    return lf_err(err, errlen, PSG_E_UNSUPPORTED_STRUCTURE,
                  "ARCE has no GPU path (the reference's ARCE does not reconstruct its blocks)");
  if ((strategy == PSG_LUPIVOT || strategy == PSG_QR) && !(tol > 0))
    return lf_err(err, errlen, PSG_E_INVALID_PARAMETER, "tol must be positive");
  int g = 1;
  if (strategy == PSG_CR) {  // cr_factor (src/localfact.cpp:266-274)
    if (blk->kind == PSG_BLOCKTRI) g = blk->m;
    else if (blk->kind == PSG_BANDED && blk->s == 1 && blk->r == 1) g = 1;
    else return lf_err(err, errlen, PSG_E_UNSUPPORTED_STRUCTURE, "cyclic reduction needs a (block) tridiagonal body");
    if (g < 1 || L % g) return lf_err(err, errlen, PSG_E_DIMENSION_MISMATCH, "body is not a whole number of blocks");
  }
  if (strategy < PSG_LU || strategy > PSG_QR) return lf_err(err, errlen, PSG_E_INVALID_PARAMETER, "unknown strategy");
  auto* h = new psg_local;
  try {
    cudaGetDevice(&h->device);
    h->stream = (cudaStream_t)stream;
    LfDev& d = h->d;
    d.strategy = strategy;
    d.L = L; d.k0 = k0; d.k1 = k1; d.es = es; d.er = er;
    d.kind = blk->kind; d.m = blk->m; d.s = blk->s; d.r = blk->r;
    d.tol = tol;
    const int w = es + 1 + er, kd = k0 + k1, dim = k0 + L + k1;
    const bool dense = strategy == PSG_LUPIVOT || strategy == PSG_QR;
    const int kdmax = dense ? dim : kd;
    Arena a;
    const size_t o_env = a.take((size_t)L * w, 8), o_b0 = a.take((size_t)L * k0, 8), o_c0 = a.take((size_t)L * k0, 8),
                 o_b1 = a.take((size_t)L * k1, 8), o_c1 = a.take((size_t)L * k1, 8), o_ar = a.take((size_t)k1 * k1, 8);
    const size_t o_z = a.take((size_t)L * k0, 8), o_w = a.take((size_t)L * k0, 8), o_y = a.take((size_t)L * k1, 8),
                 o_v = a.take((size_t)L * k1, 8), o_a1 = a.take((size_t)k0 * k0, 8), o_a2 = a.take((size_t)k1 * k1, 8),
                 o_be = a.take((size_t)k1 * k0, 8), o_ga = a.take((size_t)k0 * k1, 8),
                 o_kept = a.take((size_t)kdmax * kdmax, 8);
    const size_t o_st = a.take(ST_COUNT, 4);
    size_t o_fac = 0, o_dvec = 0, o_mu = 0, o_flag = 0;
    if (strategy == PSG_LU || strategy == PSG_LUD) {
      o_fac = a.take((size_t)L * w, 8);
      o_dvec = a.take(L, 8);
      o_mu = a.take(L, 8);
      o_flag = a.take(L, 4);
    }
    size_t o_ca = 0, o_cd = 0, o_cc = 0, o_ei = 0, o_act = 0, o_keep = 0, o_em = 0, o_d2 = 0, o_d2i = 0, o_cm = 0,
           o_rm = 0, o_rmd = 0, o_corr = 0, o_tmp = 0, o_lu = 0, o_perm = 0;
    const int nb = L / g, rg = 2 * g;
    if (strategy == PSG_CR) {
      const size_t gg = (size_t)g * g;
      o_ca = a.take(nb * gg, 8); o_cd = a.take(nb * gg, 8); o_cc = a.take(nb * gg, 8);
      o_ei = a.take(3 * (size_t)nb, 4); o_act = a.take(nb, 4); o_keep = a.take(nb, 4);
      o_em = a.take((size_t)nb * 5 * gg, 8);
      o_d2 = a.take((size_t)rg * rg, 8); o_d2i = a.take((size_t)rg * rg, 8);
      o_cm = a.take((size_t)rg * kd, 8); o_rm = a.take((size_t)kd * rg, 8); o_rmd = a.take((size_t)kd * rg, 8);
      o_corr = a.take((size_t)kd * kd, 8); o_tmp = a.take(gg, 8); o_lu = a.take((size_t)rg * rg, 8);
      o_perm = a.take(rg, 4);
    }
    size_t o_W = 0, o_Lm = 0, o_Li = 0, o_vv = 0, o_rs = 0, o_cs = 0, o_ao = 0, o_def = 0, o_kr = 0, o_kc = 0,
           o_pr = 0, o_ep = 0, o_ea = 0;
    if (dense) {
      const size_t dd = (size_t)dim * dim;
      o_W = a.take(dd, 8); o_Lm = a.take(dd, 8); o_Li = a.take(dd, 8); o_vv = a.take(dim, 8);
      o_rs = a.take(2 * (size_t)dim, 4); o_cs = a.take(dim, 4); o_ao = a.take(2 * (size_t)dim, 4);
      o_def = a.take(2 * (size_t)dim, 4); o_kr = a.take(dim, 4); o_kc = a.take(dim, 4); o_pr = a.take(dim, 4);
      o_ep = a.take(dim, 4); o_ea = a.take(dim, 8);
    }
    h->io_off = a.take(2 * (size_t)L + kdmax, 8);
    h->scr_off = a.take((size_t)std::max(dim, 4 * rg + 8), 8);
    LF_TRY(cudaMalloc(&h->base, a.bytes));
    char* B = h->base;
    auto D = [&](size_t o) { return reinterpret_cast<double*>(B + o); };
    auto I = [&](size_t o) { return reinterpret_cast<int*>(B + o); };
    d.env = D(o_env); d.b0 = D(o_b0); d.c0 = D(o_c0); d.b1 = D(o_b1); d.c1 = D(o_c1); d.ar = D(o_ar);
    d.z = D(o_z); d.w = D(o_w); d.y = D(o_y); d.v = D(o_v);
    d.a1 = D(o_a1); d.a2 = D(o_a2); d.be = D(o_be); d.ga = D(o_ga); d.kept = D(o_kept);
    d.st = I(o_st);
    if (o_fac) { d.fac = D(o_fac); d.dvec = D(o_dvec); d.mu = D(o_mu); d.flag = I(o_flag); }
    if (strategy == PSG_CR) {
      d.g = g; d.nb = nb;
      d.ca = D(o_ca); d.cd = D(o_cd); d.cc = D(o_cc); d.elim_idx = I(o_ei); d.act = I(o_act); d.keep = I(o_keep);
      d.elim_mat = D(o_em); d.d2 = D(o_d2); d.d2inv = D(o_d2i); d.cmat = D(o_cm); d.rmat = D(o_rm);
      d.rmd2 = D(o_rmd); d.corr = D(o_corr); d.tmp = D(o_tmp); d.lu = D(o_lu); d.perm = I(o_perm);
    }
    if (dense) {
      d.dim = dim;
      d.W = D(o_W); d.Lm = D(o_Lm); d.Li = D(o_Li); d.vv = D(o_vv); d.row_state = I(o_rs); d.col_state = I(o_cs);
      d.a_order = I(o_ao); d.deferred = I(o_def); d.kept_rows = I(o_kr); d.kept_cols = I(o_kc);
      d.pair_row = I(o_pr); d.ext_pos = I(o_ep); d.ext_alpha = D(o_ea);
    }
    cudaStream_t s = h->stream;
    LF_TRY(cudaMemsetAsync(B, 0, a.bytes, s));
    auto up = [&](size_t o, const double* src, size_t count) {
      if (count && src) LF_TRY(cudaMemcpyAsync(B + o, src, count * 8, cudaMemcpyHostToDevice, s));
    };
    up(o_env, blk->env, (size_t)L * w);
    up(o_b0, blk->b0, (size_t)L * k0);
    up(o_c0, blk->c0, (size_t)L * k0);
    up(o_b1, blk->b1, (size_t)L * k1);
    up(o_c1, blk->c1, (size_t)L * k1);
    up(o_ar, blk->a_right, (size_t)k1 * k1);
    if (strategy == PSG_LU || strategy == PSG_LUD) lf_banded_kernel<<<1, kThreads, 0, s>>>(d);
    else if (strategy == PSG_CR) lf_cr_kernel<<<1, kThreads, 0, s>>>(d);
    else lf_dense_kernel<<<1, kThreads, 0, s>>>(d);
    LF_TRY(cudaGetLastError());
    LF_TRY(cudaMemcpyAsync(h->st, d.st, sizeof h->st, cudaMemcpyDeviceToHost, s));
    LF_TRY(cudaStreamSynchronize(s));
    if (h->st[ST_CODE]) {
      const int code = h->st[ST_CODE] - 1;
      std::string msg = code == PSG_E_ZERO_PIVOT
                            ? (strategy == PSG_CR ? std::string("singular pivot block in cyclic reduction")
                                                  : "zero pivot at body row " + std::to_string(h->st[ST_DETAIL]))
                        : code == PSG_E_EXHAUSTED_BODY
                            ? std::string(strategy == PSG_QR ? "every column deferred; body is structurally degenerate"
                                                             : "every pivot deferred; body is structurally degenerate")
                            : std::string(errc_text(code));
      delete h;
      return lf_err(err, errlen, code, msg);
    }
    *out = h;
    return 0;
  } catch (const LfFail& f) {
    delete h;
    return lf_err(err, errlen, f.code, f.msg);
  }
}

int psg_local_query(const psg_local* h, psg_local_info* info) {
  if (!h || !info) return 1 + PSG_E_INVALID_PARAMETER;
  const LfDev& d = h->d;
  std::memset(info, 0, sizeof *info);
  info->strategy = d.strategy;
  info->L = d.L;
  info->k0 = d.k0;
  info->k1 = d.k1;
  info->env_s = d.es;
  info->env_r = d.er;
  const bool dense = d.strategy == PSG_LUPIVOT || d.strategy == PSG_QR;
  info->core = d.strategy == PSG_CR ? 2 : dense ? 3 : 1;
  info->cr_levels = h->st[ST_LEVELS];
  info->g = d.g;
  info->n_elims = h->st[ST_NELIM];
  info->n_rem = h->st[ST_NREM];
  info->dim = dense ? d.dim : d.k0 + d.L + d.k1;
  info->n_a_order = h->st[ST_NAORD];
  info->n_extras = dense ? h->st[ST_NDEF] : 0;
  info->rem[0] = h->st[ST_REM0];
  info->rem[1] = h->st[ST_REM1];
  return 0;
}

int psg_local_read(const psg_local* h, int field, void* out, size_t count, char* err, size_t errlen) {
  if (!h) return lf_err(err, errlen, PSG_E_INVALID_PARAMETER, "null handle");
  DevGuard dg(h->device);
  const LfDev& d = h->d;
  const int L = d.L, k0 = d.k0, k1 = d.k1, w = d.es + 1 + d.er, kd = h->kd(), g = d.g, gg = g * g;
  const int nel = h->st[ST_NELIM], rg = h->st[ST_NREM] * g, dim = d.dim, na = h->st[ST_NAORD], nx = h->st[ST_NDEF];
  const void* src = nullptr;
  size_t n = 0, elem = 8;
  switch (field) {
    case PSG_LF_FAC: src = d.fac; n = d.fac ? (size_t)L * w : 0; break;
    case PSG_LF_DVEC: src = d.dvec; n = d.strategy == PSG_LUD ? L : 0; break;
    case PSG_LF_Z: src = d.z; n = (size_t)L * k0; break;
    case PSG_LF_W: src = d.w; n = (size_t)L * k0; break;
    case PSG_LF_Y: src = d.y; n = (size_t)L * k1; break;
    case PSG_LF_V: src = d.v; n = (size_t)L * k1; break;
    case PSG_LF_ALPHA1: src = d.a1; n = (size_t)k0 * k0; break;
    case PSG_LF_ALPHA2: src = d.a2; n = (size_t)k1 * k1; break;
    case PSG_LF_BETA: src = d.be; n = (size_t)k1 * k0; break;
    case PSG_LF_GAMMA: src = d.ga; n = (size_t)k0 * k1; break;
    case PSG_LF_KEPT: src = d.kept; n = (size_t)kd * kd; break;
    case PSG_LF_CR_ELIM_IDX: src = d.elim_idx; n = 3 * (size_t)nel; elem = 4; break;
    case PSG_LF_CR_ELIM_MAT: src = d.elim_mat; n = (size_t)nel * 5 * gg; break;
    case PSG_LF_CR_D2: src = d.d2; n = (size_t)rg * rg; break;
    case PSG_LF_CR_D2INV: src = d.d2inv; n = (size_t)rg * rg; break;
    case PSG_LF_CR_CMAT: src = d.cmat; n = (size_t)rg * kd; break;
    case PSG_LF_CR_RMAT_D2INV: src = d.rmd2; n = (size_t)kd * rg; break;
    case PSG_LF_WMID: src = d.W; n = d.W ? (size_t)dim * dim : 0; break;
    case PSG_LF_LMAT: src = d.Lm; n = d.W ? (size_t)dim * dim : 0; break;
    case PSG_LF_LINV: src = d.Li; n = d.W ? (size_t)dim * dim : 0; break;
    case PSG_LF_A_ORDER: src = d.a_order; n = 2 * (size_t)na; elem = 4; break;
    case PSG_LF_KEPT_ROWS: src = d.kept_rows; n = d.W ? kd : 0; elem = 4; break;
    case PSG_LF_KEPT_COLS: src = d.kept_cols; n = d.W ? kd : 0; elem = 4; break;
    case PSG_LF_EXTRA_POS: src = d.ext_pos; n = nx; elem = 4; break;
    case PSG_LF_EXTRA_ALPHA: src = d.ext_alpha; n = nx; break;
    default: return lf_err(err, errlen, PSG_E_INVALID_PARAMETER, "unknown field");
  }
  if (n == 0 || !src) return 0;
  if (count < n) return lf_err(err, errlen, PSG_E_DIMENSION_MISMATCH, "output too small");
  if (cudaMemcpy(out, src, n * elem, cudaMemcpyDeviceToHost) != cudaSuccess)
    return lf_err(err, errlen, PSG_E_CUDA, "cudaMemcpy failed");
  return 0;
}

namespace {

int run_op(const psg_local* h, int op, const double* body, const double* kept, double* out_body, double* out_kept,
           char* err, size_t errlen) {
  if (!h) return lf_err(err, errlen, PSG_E_INVALID_PARAMETER, "null handle");
  DevGuard dg(h->device);
  try {
    const int L = h->d.L, kd = h->kd();
    double* io = reinterpret_cast<double*>(h->base + h->io_off);
    double* scr = reinterpret_cast<double*>(h->base + h->scr_off);
    cudaStream_t s = h->stream;
    LF_TRY(cudaMemcpyAsync(io, body, sizeof(double) * L, cudaMemcpyHostToDevice, s));
    if (kept && kd) LF_TRY(cudaMemcpyAsync(io + L, kept, sizeof(double) * kd, cudaMemcpyHostToDevice, s));
    lf_op_kernel<<<1, kThreads, 0, s>>>(h->d, op, io, scr);
    LF_TRY(cudaGetLastError());
    LF_TRY(cudaMemcpyAsync(out_body, io + L + kd, sizeof(double) * L, cudaMemcpyDeviceToHost, s));
    if (out_kept && kd) LF_TRY(cudaMemcpyAsync(out_kept, io + L, sizeof(double) * kd, cudaMemcpyDeviceToHost, s));
    LF_TRY(cudaStreamSynchronize(s));
    return 0;
  } catch (const LfFail& f) {
    return lf_err(err, errlen, f.code, f.msg);
  }
}

}  // namespace

int psg_local_condense(const psg_local* h, const double* f_body, double* ghat, double* kept_rhs, char* err,
                       size_t errlen) {
  return run_op(h, OP_CONDENSE, f_body, nullptr, ghat, kept_rhs, err, errlen);
}

int psg_local_backsolve(const psg_local* h, const double* ghat, const double* x_kept, double* x, char* err,
                        size_t errlen) {
  return run_op(h, OP_BACKSOLVE, ghat, x_kept, x, nullptr, err, errlen);
}

int psg_local_apply(const psg_local* h, int which, const double* rhs, double* out, char* err, size_t errlen) {
  if (which != 0 && which != 1) return lf_err(err, errlen, PSG_E_INVALID_PARAMETER, "which must be 0 or 1");
  return run_op(h, which == 0 ? OP_NINV : OP_SINV, rhs, nullptr, out, nullptr, err, errlen);
}

void psg_local_release(psg_local* h) {
  if (!h) return;
  DevGuard dg(h->device);
  delete h;
}

int psg_dense_solve(int n, const double* T, const double* rhs, double* x, long long* ops, void* stream, char* err,
                    size_t errlen) {
  if (n < 0) return lf_err(err, errlen, PSG_E_DIMENSION_MISMATCH, "reduced rhs length");
  if (n == 0) {
    if (ops) *ops = 0;
    return 0;
  }
  cudaStream_t s = (cudaStream_t)stream;
  char* base = nullptr;
  try {
    const size_t nn = (size_t)n * n;
    const size_t bytes = nn * 8 + 2 * (size_t)n * 8 + (size_t)n * 4 + 16;
    LF_TRY(cudaMalloc(&base, bytes));
    double* lu = reinterpret_cast<double*>(base);
    double* dr = lu + nn;
    double* dx = dr + n;
    int* perm = reinterpret_cast<int*>(dx + n);
    int* bad = perm + n;
    LF_TRY(cudaMemcpyAsync(lu, T, nn * 8, cudaMemcpyHostToDevice, s));
    LF_TRY(cudaMemcpyAsync(dr, rhs, (size_t)n * 8, cudaMemcpyHostToDevice, s));
    ds_iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(perm, n, bad);
    for (int c = 0; c < n; ++c) {
      ds_pivot_kernel<<<1, 1024, 0, s>>>(lu, perm, n, c, bad);
      const size_t m = (size_t)(n - c - 1) * (n - c - 1);
      if (m) ds_update_kernel<<<(unsigned)std::min<size_t>((m + 255) / 256, 4 * 148), 256, 0, s>>>(lu, n, c, bad);
    }
    ds_subst_kernel<<<1, 32, 0, s>>>(lu, perm, n, dr, dx, bad);
    LF_TRY(cudaGetLastError());
    int hbad = 0;
    LF_TRY(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s));
    LF_TRY(cudaMemcpyAsync(x, dx, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    LF_TRY(cudaStreamSynchronize(s));
    cudaFree(base);
    base = nullptr;
    if (hbad) return lf_err(err, errlen, PSG_E_SINGULAR_REDUCED_SYSTEM, "reduced system is singular");
    if (ops) {  // multiply-adds the reference counts (src/parfact.cpp:142-181)
      long long c = 0;
      for (long long q = 0; q < n; ++q) c += (n - 1 - q) * (n - q);
      *ops = c + (long long)n * (n - 1) + n;
    }
    return 0;
  } catch (const LfFail& f) {
    if (base) cudaFree(base);
    return lf_err(err, errlen, f.code, f.msg);
  }
}

}  // extern "C"
