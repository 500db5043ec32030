// psg_common.cuh -- device-side helpers shared by the partition-solver
// kernels: row-array views of the reference storage, TMA bulk staging with
// mbarriers (cp.async.bulk, sm_90+/sm_100a), status words.
#pragma once
#include <climits>

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
  int lo, hi;    // rows with a defined value (outside: structural zero)
  long slo, shi; // rows whose address lies inside the allocation (safe to over-read)
};

__host__ __device__ inline RowArr make_rows(const double* p, int lo, int hi, long slo, long shi) {
  return RowArr{p, lo, hi, slo, shi};
}
__host__ __device__ inline RowArr make_rows(const double* p, int lo, int hi) { return RowArr{p, lo, hi, lo, hi}; }

__device__ __forceinline__ double row_at(const RowArr& X, long r) {
  return (r >= X.lo && r < X.hi) ? __ldg(X.p + r) : 0.0;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Device status shared by all kernels of one solve.  The certificate max is
// spread over kCertSlots words (by block index) to keep same-address atomic
// traffic low when every CTA reports; the host takes the max of the slots.
constexpr int kCertSlots = 32;
struct DevStatus {
  unsigned long long cert_bits[kCertSlots];  // max componentwise backward error (double bits, >= 0)
  int bad_seg;                               // lowest segment with a non-finite solution value (INT_MAX: none)
  int pivot_seg;                             // lowest segment whose own elimination hit a zero/non-finite pivot
};

__device__ __forceinline__ void status_nonfinite(DevStatus* st, int seg) { atomicMin(&st->bad_seg, seg); }
__device__ __forceinline__ void status_pivot(DevStatus* st, int seg) { atomicMin(&st->pivot_seg, seg); }

__device__ __forceinline__ void status_cert(DevStatus* st, double w) {
  if (!(w <= 1.0e300)) w = __longlong_as_double(0x7ff0000000000000ll);  // NaN/huge -> +inf
  atomicMax(&st->cert_bits[blockIdx.x % kCertSlots], (unsigned long long)__double_as_longlong(w));
}

__device__ __forceinline__ void status_reset(DevStatus* st) {
  for (int k = 0; k < kCertSlots; ++k) st->cert_bits[k] = 0ull;
  st->bad_seg = INT_MAX;
  st->pivot_seg = INT_MAX;
}

// The last block of the grid to get here publishes the solve's status straight
// into the caller's pinned host slot (no device-to-host copy in the stream);
// every thread of every block calls it after its last status update, done_ctr
// (zero before the launch) resets itself.
__device__ __forceinline__ void status_publish_last(DevStatus* st, DevStatus* host_out, unsigned* done_ctr) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(st);
  volatile unsigned long long* dst = reinterpret_cast<volatile unsigned long long*>(host_out);
  for (int i = threadIdx.x; i < (int)(sizeof(DevStatus) / 8); i += blockDim.x)
    dst[i] = atomicAdd(const_cast<unsigned long long*>(src + i), 0ull);  // coherent read of the atomically-updated words
  if (threadIdx.x == 0) *done_ctr = 0u;
  __threadfence_system();
}

// cp.async (LDGSTS) 8-byte copy global -> shared, no register staging.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// cp.async 16-byte copy global -> shared (L2 only), per-thread commit groups
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine, non-tensor form)
// ---------------------------------------------------------------------------


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

// Stage rows [r0, r1) of X into shared memory: issue side.  `base` must be
// 16-byte aligned with room for (r1 - r0 + 3) doubles; the result buffer is
// buf = base + 1 + shift (shift 0/1) with buf[r - r0] = row r, buf[j] and row
// r0+j congruent mod 16 bytes.  The copy is widened to 16-byte boundaries when
// the widened bytes stay inside the allocation (X.slo/X.shi), so in the
// common case a single bulk copy moves everything and nothing blocks; rows
// outside X's defined range are zeroed afterwards by stage_fixup.  Returns
// shift; *tx accumulates the bulk bytes.  Called by one lane per array.
__device__ __forceinline__ int stage_issue(const RowArr& X, long r0, long r1, double* base, uint64_t* bar,
                                           uint32_t* tx) {
  const uintptr_t g0 = reinterpret_cast<uintptr_t>(X.p + r0);
  const uintptr_t s0 = reinterpret_cast<uintptr_t>(base + 1);
  const int shift = (int)(((g0 - s0) >> 3) & 1);
  double* buf = base + 1 + shift;
  long v0 = r0 > X.lo ? r0 : X.lo;
  long v1 = r1 < X.hi ? r1 : X.hi;
  if (v1 <= v0) return shift;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(X.p + v0);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(X.p + v1);
  uintptr_t b0 = a0 & ~uintptr_t(15), b1 = (a1 + 15) & ~uintptr_t(15);
  const bool head_ok = (long)(v0 - ((a0 - b0) >> 3)) >= X.slo;
  const bool tail_ok = (long)(v1 + ((b1 - a1) >> 3)) <= X.shi;
  if (!head_ok) b0 = (a0 + 15) & ~uintptr_t(15);
  if (!tail_ok) b1 = a1 & ~uintptr_t(15);
  if (b1 > b0) {
    const long rb = v0 + ((long)b0 - (long)a0) / 8;
    bulk_g2s(buf + (rb - r0), reinterpret_cast<const void*>(b0), (uint32_t)(b1 - b0), bar);
    *tx += (uint32_t)(b1 - b0);
    if (!head_ok && a0 < b0) buf[v0 - r0] = __ldg(X.p + v0);
    if (!tail_ok && a1 > b1) buf[v1 - 1 - r0] = __ldg(X.p + v1 - 1);
  } else {
    for (long r = v0; r < v1; ++r) buf[r - r0] = __ldg(X.p + r);
  }
  return shift;
}

// After the mbarrier wait: zero the staged rows that lie outside X's defined
// range (only the first/last segments of an array have any).
__device__ __forceinline__ void stage_fixup(const RowArr& X, long r0, long r1, double* buf) {
  for (long r = r0; r < r1 && r < X.lo; ++r) buf[r - r0] = 0.0;
  for (long r = (X.hi > r0 ? X.hi : r0); r < r1; ++r) buf[r - r0] = 0.0;
}

// Bulk shared->global copy (async proxy); dst/src 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_and_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32-byte aligned load of 4 doubles (one LDG.256: one sector per request
// instead of four for a lane walking its own contiguous rows)
__device__ __forceinline__ void ldg256(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// L2 eviction-priority policies (createpolicy) and the hinted 256-bit forms:
// streamed-once data evict_first, a scratch written and read back soon evict_last
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void ldg256h(const double* p, unsigned long long pol, double& a, double& b, double& c,
                                        double& d) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
      : "l"(p), "l"(pol));
}
__device__ __forceinline__ void stg256h(double* p, unsigned long long pol, double a, double b, double c, double d) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void stg256(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// Reciprocal: MUFU approximation + two Newton steps (<= 1 ulp; no slow-path
// branch).  0 -> inf and inf/NaN -> NaN propagate to the non-finite check.
// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start before its predecessor in
// the stream has finished; pdl_wait() blocks until the predecessor's writes
// are visible, pdl_trigger() lets the successor's CTAs launch early.  Both are
// no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Host-visible launch accounting.
struct LaunchCounter {
  int n = 0;
  void add(int k = 1) { n += k; }
};

}  // namespace psg
