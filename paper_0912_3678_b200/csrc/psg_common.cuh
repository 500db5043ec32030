// psg_common.cuh -- device-side helpers shared by the partition-solver
// kernels: row-array views of the reference storage, TMA bulk staging with
// mbarriers (cp.async.bulk, sm_90+/sm_100a), status words.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace psg {

// A "row array": element for matrix row r lives at p[r] and is defined for
// lo <= r < hi (outside: structural zero).  This is how the kernels address
// the reference layouts without copying them: e.g. the tridiagonal
// sub-diagonal a_r = data[r-1] is {data - 1, 1, n}, the diagonal
// b_r = data[n-1+r] is {data + n - 1, 0, n} (src/structmat.cpp:33-38).
struct RowArr {
  const double* p;
  int lo, hi;
};

__device__ __forceinline__ double row_at(const RowArr& X, long r) {
  return (r >= X.lo && r < X.hi) ? __ldg(X.p + r) : 0.0;
}

// Device status shared by all kernels of one solve.
struct DevStatus {
  unsigned long long cert_bits;  // max componentwise backward error (double bits, >= 0)
  int bad_seg;                   // lowest segment with a non-finite value (INT_MAX: none)
  int pad;
};

__device__ __forceinline__ void status_nonfinite(DevStatus* st, int seg) { atomicMin(&st->bad_seg, seg); }

__device__ __forceinline__ void status_cert(DevStatus* st, double w) {
  if (!(w <= 1.0e300)) w = __longlong_as_double(0x7ff0000000000000ll);  // NaN/huge -> +inf
  atomicMax(&st->cert_bits, (unsigned long long)__double_as_longlong(w));
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine, non-tensor form)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// Bulk global->shared copy; dst/src 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Stage rows [r0, r1) of X into shared memory.  `base` must be 16-byte
// aligned with room for (r1 - r0 + 1) doubles.  Returns buf with
// buf[r - r0] = X(r) (zero outside X's valid range).  The 16-byte aligned
// interior goes through one bulk copy (counted into *tx); the <= 2 ragged
// elements at either end and the zero fill are plain shared stores.  Must be
// called by ONE thread; the caller publishes with __syncthreads + mbar wait.
__device__ __forceinline__ double* stage_rows(const RowArr& X, long r0, long r1, double* base,
                                              uint64_t* bar, uint32_t* tx) {
  const uintptr_t g0 = reinterpret_cast<uintptr_t>(X.p + r0);
  const uintptr_t s0 = reinterpret_cast<uintptr_t>(base);
  const int shift = (int)(((g0 - s0) >> 3) & 1);  // make buf[j] and row r0+j congruent mod 16
  double* buf = base + shift;
  const long v0 = r0 > X.lo ? r0 : X.lo;
  const long v1 = r1 < X.hi ? r1 : X.hi;
  for (long r = r0; r < r1 && r < v0; ++r) buf[r - r0] = 0.0;
  for (long r = (v1 > r0 ? v1 : r0); r < r1; ++r) buf[r - r0] = 0.0;
  if (v1 <= v0) return buf;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(X.p + v0);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(X.p + v1);
  const uintptr_t b0 = (a0 + 15) & ~uintptr_t(15);
  const uintptr_t b1 = a1 & ~uintptr_t(15);
  if (b1 > b0) {
    const long rb = v0 + (long)((b0 - a0) >> 3);
    bulk_g2s(buf + (rb - r0), reinterpret_cast<const void*>(b0), (uint32_t)(b1 - b0), bar);
    *tx += (uint32_t)(b1 - b0);
    if (a0 < b0) buf[v0 - r0] = __ldg(X.p + v0);
    if (a1 > b1) buf[v1 - 1 - r0] = __ldg(X.p + v1 - 1);
  } else {
    for (long r = v0; r < v1; ++r) buf[r - r0] = __ldg(X.p + r);
  }
  return buf;
}

// Host-visible launch accounting.
struct LaunchCounter {
  int n = 0;
  void add(int k = 1) { n += k; }
};

}  // namespace psg
