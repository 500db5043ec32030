// gen_kernels.cuh -- device generator of the BASELINE config instances
// (SplitMix64 counter draws, bit-identical to parsol::SplitMix64,
// include/parsol/rng.hpp:11-35, and to oracle or_generate_config) and the
// device matvec / residual (src/structmat.cpp:211-269, src/parfact.cpp:241-251).
#pragma once

#include "psg_common.cuh"

namespace psg {

__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// (k+1)-th draw of (seed, stream) mapped to (-1, 1) exactly like next_unit().
__device__ __forceinline__ double sm_unit(uint64_t seed, uint64_t stream, uint64_t e) {
  const uint64_t base = sm_mix(seed + 0x9E3779B97F4A7C15ull * (stream + 1));
  const uint64_t u = sm_mix(base + 0x9E3779B97F4A7C15ull * (e + 1)) >> 11;
  return __dadd_rn(__dadd_rn(__dmul_rn(2.0, __ddiv_rn((double)u, 9007199254740992.0)), -1.0),
                   1.1102230246251565e-16);
}

// U[0,1] = (unit+1)/2 ; U[-1/2,1/2] = unit/2
__device__ __forceinline__ double u01(uint64_t seed, uint64_t st, uint64_t e) {
  return __dmul_rn(0.5, __dadd_rn(sm_unit(seed, st, e), 1.0));
}
__device__ __forceinline__ double uhalf(uint64_t seed, uint64_t st, uint64_t e) {
  return __dmul_rn(0.5, sm_unit(seed, st, e));
}

// cfg 0/1: data = [sub (n-1) | diag (n) | super (n-1)], f
__global__ void gen_tridiag_kernel(uint64_t seed, int n, double* data, double* f) {
  const long total = 3L * n - 2;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total + n; e += (long)gridDim.x * blockDim.x) {
    if (e < n - 1) {
      data[e] = sm_unit(seed, 0, e);
    } else if (e < 2L * n - 1) {
      const long t = e - (n - 1);
      data[e] = __dadd_rn(4.0, u01(seed, 1, t));
    } else if (e < total) {
      data[e] = sm_unit(seed, 2, e - (2L * n - 1));
    } else {
      f[e - total] = sm_unit(seed, 3, e - total);
    }
  }
}

// cfg 2: block tridiagonal m = 4, N block rows; storage per block row b:
// [sub | diag | super] at offset (3b-1)*16 (b > 0).
__global__ void gen_blocktri_kernel(uint64_t seed, int N, double* data, double* f) {
  const long total = (3L * N - 2) * 16;
  const long n = 4L * N;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total + n; e += (long)gridDim.x * blockDim.x) {
    if (e >= total) {
      f[e - total] = sm_unit(seed, 3, e - total);
      continue;
    }
    // locate block row: row 0 has 32 entries, others 48 (the last has 32).
    long b, within;
    if (e < 32) {
      b = 0;
      within = e + 16;  // pretend a sub block precedes
    } else {
      b = (e - 32) / 48 + 1;
      within = e - (3 * b - 1) * 16;
    }
    const int blk = (int)(within / 16), t = (int)(within % 16);
    double v;
    if (blk == 0)
      v = uhalf(seed, 1, (b - 1) * 16 + t);
    else if (blk == 1)
      v = __dadd_rn((t / 4 == t % 4) ? 8.0 : 0.0, uhalf(seed, 0, b * 16 + t));
    else
      v = uhalf(seed, 2, b * 16 + t);
    data[e] = v;
  }
}

// cfg 3: banded s = r = 3: bands d = -3..3, band d holds n-|d| entries.
__global__ void gen_banded7_kernel(uint64_t seed, int n, double* data, double* f) {
  const long total = 7L * n - 12;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total + n; e += (long)gridDim.x * blockDim.x) {
    if (e >= total) {
      f[e - total] = sm_unit(seed, 2, e - total);
      continue;
    }
    long pos = 0, offd = 0;
    int d = -3;
    for (; d <= 3; ++d) {
      const long len = n - (d < 0 ? -d : d);
      if (e < pos + len) break;
      pos += len;
      if (d != 0) offd += len;
    }
    const long t = e - pos;
    data[e] = (d == 0) ? __dadd_rn(8.0, u01(seed, 1, t)) : sm_unit(seed, 0, offd + t);
  }
}

// cfg 4: BABD m = 8, s = 8, r = 0, N intervals, BC row first.
__global__ void gen_babd_kernel(uint64_t seed, int N, double* data, double* corner, double* f) {
  const long total = 64 + 128L * N;
  const long n = 8L * (N + 1);
  const double hh = __dmul_rn(0.5, __ddiv_rn(1.0, (double)N));
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total + n + 64; e += (long)gridDim.x * blockDim.x) {
    if (e < 64) {
      data[e] = (e / 8 == e % 8) ? 1.0 : 0.0;
    } else if (e < total) {
      const long k = (e - 64) / 128;
      const int w = (int)((e - 64) % 128), i = w / 16, jj = w % 16;
      const double id = (i == (jj % 8)) ? 1.0 : 0.0;
      if (jj < 8) {
        const double mk = __ddiv_rn(sm_unit(seed, 0, k * 64 + i * 8 + jj), 8.0);
        data[e] = -__dadd_rn(id, __dmul_rn(hh, mk));
      } else {
        const double mk1 = __ddiv_rn(sm_unit(seed, 0, (k + 1) * 64 + i * 8 + (jj - 8)), 8.0);
        data[e] = __dsub_rn(id, __dmul_rn(hh, mk1));
      }
    } else if (e < total + n) {
      const long r = e - total;
      if (r < 8) {
        f[r] = sm_unit(seed, 3, r);
      } else {
        const long k = (r - 8) / 8;
        const int i = (int)((r - 8) % 8);
        f[r] = __dmul_rn(hh, __dadd_rn(sm_unit(seed, 1, k * 8 + i), sm_unit(seed, 1, (k + 1) * 8 + i)));
      }
    } else {
      corner[e - total - n] = uhalf(seed, 2, e - total - n);
    }
  }
}

// ----------------------------------------------------------------------------
// matvec / residual with the reference's ascending-column order and no FMA
// contraction (for_each_in_row, src/structmat.cpp:211-248).
// ----------------------------------------------------------------------------
struct MatView {
  int kind, n, m, s, r;
  const double* data;
  const double* corner;
  int cr, cc;
};

__device__ __forceinline__ long band_off(int n, int s, int d) {
  // sum_{b=-s}^{d-1} (n - |b|)
  long off = 0;
  for (int b = -s; b < d; ++b) off += n - (b < 0 ? -b : b);
  return off;
}

__device__ double row_dot(const MatView& A, long i, const double* __restrict__ x) {
  double acc = 0.0;
  const int n = A.n, m = A.m;
  if (A.kind == 0) {  // banded
    const long j0 = i - A.s > 0 ? i - A.s : 0;
    const long j1 = i + A.r < n - 1 ? i + A.r : n - 1;
    for (long j = j0; j <= j1; ++j) {
      const int d = (int)(j - i);
      const long i0 = d < 0 ? -d : 0;
      acc = __dadd_rn(acc, __dmul_rn(A.data[band_off(n, A.s, d) + (i - i0)], x[j]));
    }
  } else if (A.kind == 1) {  // block tridiagonal
    const long bi = i / m;
    const long off = bi == 0 ? 0 : (3 * bi - 1) * (long)m * m;
    const long j0 = (bi - 1) * m > 0 ? (bi - 1) * m : 0;
    const long j1 = (bi + 2) * m < n ? (bi + 2) * m : n;
    for (long j = j0; j < j1; ++j) {
      const long bj = j / m;
      const long blk = bi > 0 ? bj - bi + 1 : bj - bi;
      acc = __dadd_rn(acc, __dmul_rn(A.data[off + blk * m * m + (i - bi * m) * m + (j - bj * m)], x[j]));
    }
  } else if (A.kind == 4) {  // circulant-like: columns (i + d) mod n, ascending (src/structmat.cpp:234-245)
    for (int d = -A.s; d <= A.r; ++d)  // wrapped past the end: smallest columns
      if (i + d >= n) acc = __dadd_rn(acc, __dmul_rn(A.data[(long)(d + A.s) * n + i], x[i + d - n]));
    for (int d = -A.s; d <= A.r; ++d)
      if (i + d >= 0 && i + d < n) acc = __dadd_rn(acc, __dmul_rn(A.data[(long)(d + A.s) * n + i], x[i + d]));
    for (int d = -A.s; d <= A.r; ++d)  // wrapped before the start: largest columns
      if (i + d < 0) acc = __dadd_rn(acc, __dmul_rn(A.data[(long)(d + A.s) * n + i], x[i + d + n]));
  } else {  // abd / babd: closed-form block-row offsets
    const long b = i / m;
    const long c0 = b * m - A.s > 0 ? b * m - A.s : 0;
    const long c1 = b * m + m + A.r < n ? b * m + m + A.r : n;
    const long off = b == 0 ? 0 : (long)m * (m + A.r) + (b - 1) * (long)m * (m + A.r + A.s);
    const long w = c1 - c0;
    for (long j = c0; j < c1; ++j) acc = __dadd_rn(acc, __dmul_rn(A.data[off + (i - b * m) * w + (j - c0)], x[j]));
    if (A.kind == 3 && i < A.cr)
      for (long j = n - A.cc; j < n; ++j)
        acc = __dadd_rn(acc, __dmul_rn(A.corner[i * A.cc + (j - (n - A.cc))], x[j]));
  }
  return acc;
}

__global__ void matvec_kernel(MatView A, const double* __restrict__ x, double* __restrict__ y) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < A.n; i += (long)gridDim.x * blockDim.x)
    y[i] = row_dot(A, i, x);
}

// out[0] = max |Ax - f| bits, out[1] = max |f| bits  (non-negative doubles
// compare like their bit patterns; NaN is mapped to +inf).
__global__ void residual_kernel(MatView A, const double* __restrict__ x, const double* __restrict__ f,
                                unsigned long long* out) {
  double num = 0.0, den = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < A.n; i += (long)gridDim.x * blockDim.x) {
    double v = fabs(__dsub_rn(row_dot(A, i, x), f[i]));
    if (!(v <= 1.0e308)) v = __longlong_as_double(0x7ff0000000000000ll);
    num = fmax(num, v);
    den = fmax(den, fabs(f[i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    num = fmax(num, __shfl_xor_sync(0xffffffffu, num, o));
    den = fmax(den, __shfl_xor_sync(0xffffffffu, den, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out + 0, (unsigned long long)__double_as_longlong(num));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(den));
  }
}

// r = f - A x (no FMA, ascending columns) and out[0] = max|r| bits, out[1] = max|f| bits.
__global__ void residual_vec_kernel(MatView A, const double* __restrict__ x, const double* __restrict__ f,
                                    double* __restrict__ r, unsigned long long* out) {
  double num = 0.0, den = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < A.n; i += (long)gridDim.x * blockDim.x) {
    const double ri = __dsub_rn(f[i], row_dot(A, i, x));
    r[i] = ri;
    double v = fabs(ri);
    if (!(v <= 1.0e308)) v = __longlong_as_double(0x7ff0000000000000ll);
    num = fmax(num, v);
    den = fmax(den, fabs(f[i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    num = fmax(num, __shfl_xor_sync(0xffffffffu, num, o));
    den = fmax(den, __shfl_xor_sync(0xffffffffu, den, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out + 0, (unsigned long long)__double_as_longlong(num));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(den));
  }
}

__global__ void axpy_kernel(long n, const double* __restrict__ d, double* __restrict__ x) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) x[i] += d[i];
}

}  // namespace psg
