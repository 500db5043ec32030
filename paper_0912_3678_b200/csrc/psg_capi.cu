// psg_capi.cu -- the C ABI (include/psg.h) of the B200 partition solver:
// descriptor validation, partition planning, handle/buffer ownership and the
// launch sequences of the factor / solve phases.
//
// Single translation unit: the kernels live in the *.cuh headers included
// below, all compiled for sm_100a only.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/psg.h"
#include "gen_exact.cuh"
#include "gen_kernels.cuh"
#include "psg_common.cuh"
#include "tri_kernels.cuh"
#include "blk_kernels.cuh"
#include "band_kernels.cuh"
#include "chain_kernels.cuh"
#include "ode_kernels.cuh"
#include "piv_kernels.cuh"
#include "pr_kernels.cuh"

using namespace psg;

namespace {

// ----------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------
struct Fail {
  int code;  // psg_errc
  std::string msg;
};

double bits_to_double(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}

int set_err(char* err, size_t errlen, int code, const std::string& msg) {
  if (err && errlen) {
    std::snprintf(err, errlen, "%s", msg.c_str());
  }
  return 1 + code;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      throw Fail{PSG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)};            \
  } while (0)

#define LAUNCH_CHECK() CUDA_TRY(cudaGetLastError())

// A handle's buffers live on the device it was factored on: every entry
// point that takes a handle runs there and restores the caller's device.
struct DeviceGuard {
  int prev = -1, want = -1;
  explicit DeviceGuard(int d) : want(d) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor drains and calls pdl_wait() before consuming its output.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, args...));
}

// The dynamic shared memory opt-in is a per-device attribute: set it once per
// (kernel, device), also for processes that drive several GPUs.
void ensure_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (done.count({kernel, dev})) return;
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({kernel, dev});
}

// Process-wide cache of device blocks keyed by byte size: repeated
// parallel_factor calls on same-shaped systems reuse memory instead of
// paying cudaMalloc (and its implicit device synchronisation) each time.
// Blocks are returned only after the owning handle's work has completed.
// Device buffers are recycled by exact size (a handle re-created per step,
// as the drop-in path does, costs no cudaMalloc/cudaFree), keyed by device.
// At most kCacheCap bytes stay cached; an allocation that fails with
// out-of-memory flushes the cache and retries.
struct BlockCache {
  static constexpr size_t kCacheCap = size_t(8) << 30;
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free_;
  size_t cached = 0;
  static int device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
  }
  void flush() {
    std::lock_guard<std::mutex> g(mu);
    int cur = device();
    for (auto& kv : free_) {
      cudaSetDevice(kv.first.first);
      cudaFree(kv.second);
    }
    cudaSetDevice(cur);
    free_.clear();
    cached = 0;
  }
  void* get(size_t bytes) {
    const int dev = device();
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = free_.find({dev, bytes});
      if (it != free_.end()) {
        void* p = it->second;
        free_.erase(it);
        cached -= bytes;
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();  // clear the sticky-free error state of the failed call
      flush();
      e = cudaMalloc(&p, bytes);
    }
    CUDA_TRY(e);
    return p;
  }
  void put(void* p, size_t bytes, int dev) {
    {
      std::lock_guard<std::mutex> g(mu);
      if (cached + bytes <= kCacheCap) {
        free_.emplace(std::make_pair(dev, bytes), p);
        cached += bytes;
        return;
      }
    }
    int cur = device();
    cudaSetDevice(dev);
    cudaFree(p);
    cudaSetDevice(cur);
  }
};

BlockCache& block_cache() {
  static BlockCache* c = new BlockCache;  // intentionally leaked (outlives static dtors)
  return *c;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0, bytes = 0;
  int dev = 0;  // device the buffer lives on
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) block_cache().put(p, bytes, dev);
    p = nullptr;
    n = bytes = 0;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    reset();
    bytes = ((sizeof(T) * std::max<size_t>(count, 1)) + 511) & ~size_t(511);
    dev = BlockCache::device();
    p = static_cast<T*>(block_cache().get(bytes));
    n = count;
  }
};

// Small pinned host slots (status words) carved from one page-locked slab.
struct PinnedSlots {
  std::mutex mu;
  char* slab = nullptr;
  std::vector<int> free_;
  static constexpr int kSlot = 512, kCount = 256;
  void* get() {
    std::lock_guard<std::mutex> g(mu);
    if (!slab) {
      CUDA_TRY(cudaMallocHost(&slab, kSlot * kCount));
      for (int i = kCount - 1; i >= 0; --i) free_.push_back(i);
    }
    if (free_.empty()) throw Fail{PSG_E_CUDA, "out of pinned status slots"};
    int i = free_.back();
    free_.pop_back();
    return slab + (size_t)i * kSlot;
  }
  void put(void* p) {
    std::lock_guard<std::mutex> g(mu);
    free_.push_back(int((static_cast<char*>(p) - slab) / kSlot));
  }
};

PinnedSlots& pinned_slots() {
  static PinnedSlots* s = new PinnedSlots;
  return *s;
}

// ----------------------------------------------------------------------------
// descriptor validation: make() (src/structmat.cpp:153-207), with the Babd
// s = m, r = 0 relaxation the BVP config needs.
// ----------------------------------------------------------------------------
size_t body_entry_count(int kind, long n, long m, long s, long r) {  // src/structmat.cpp:64-84
  switch (kind) {
    case PSG_BANDED: {
      size_t c = 0;
      for (long d = -s; d <= r; ++d) c += size_t(n - std::labs(d));
      return c;
    }
    case PSG_BLOCKTRI: return size_t(3 * (n / m) - 2) * m * m;
    case PSG_ABD:
    case PSG_BABD: {
      const long nb = n / m;
      size_t off = 0;
      for (long q = 0; q < nb; ++q) {
        const long c0 = std::max(0L, q * m - s), c1 = std::min(n, q * m + m + r);
        off += size_t(m) * (c1 - c0);
      }
      return off;
    }
    case PSG_CIRCULANT: return size_t(s + r + 1) * n;
  }
  return 0;
}

void validate(const psg_desc& A) {
  const int n = A.n, m = A.m, s = A.s, r = A.r;
  if (n <= 0) throw Fail{PSG_E_DIMENSION_MISMATCH, "n must be positive"};
  if (m <= 0) throw Fail{PSG_E_DIMENSION_MISMATCH, "m must be positive"};
  if (s < 0 || r < 0) throw Fail{PSG_E_INVALID_BANDWIDTH, "bandwidths must be non-negative"};
  switch (A.kind) {
    case PSG_BANDED:
    case PSG_CIRCULANT:
      if (m != 1) throw Fail{PSG_E_DIMENSION_MISMATCH, "scalar kinds require m = 1"};
      if (s + r + 1 > n) throw Fail{PSG_E_INVALID_BANDWIDTH, "band wider than matrix"};
      break;
    case PSG_BLOCKTRI:
      if (n % m != 0) throw Fail{PSG_E_DIMENSION_MISMATCH, "n must be a multiple of m"};
      if (s != 1 || r != 1) throw Fail{PSG_E_INVALID_BANDWIDTH, "block tridiagonal requires s = r = 1"};
      break;
    case PSG_ABD:
    case PSG_BABD: {
      if (n % m != 0) throw Fail{PSG_E_DIMENSION_MISMATCH, "n must be a multiple of m"};
      if (m < 2) throw Fail{PSG_E_DIMENSION_MISMATCH, "ABD requires m >= 2"};
      const bool ok = (s >= 1 && r >= 1 && s + r == m) || (A.kind == PSG_BABD && s == m && r == 0);
      if (!ok) throw Fail{PSG_E_INVALID_BANDWIDTH, "ABD requires s,r >= 1 with s + r = m (Babd also s = m, r = 0)"};
      if (n / m < 2) throw Fail{PSG_E_DIMENSION_MISMATCH, "ABD requires at least 2 block rows"};
      break;
    }
    default: throw Fail{PSG_E_UNSUPPORTED_KIND, "unknown kind"};
  }
  if (A.kind == PSG_BABD) {
    if (!A.corner) throw Fail{PSG_E_DIMENSION_MISMATCH, "BABD requires a corner block"};
    if (A.corner_rows < 1 || A.corner_cols < 1 || A.corner_rows > m || A.corner_cols > m)
      throw Fail{PSG_E_DIMENSION_MISMATCH, "corner block must fit inside the first/last block"};
    if (m + r > n - A.corner_cols) throw Fail{PSG_E_DIMENSION_MISMATCH, "corner overlaps the first block row span"};
  } else if (A.corner || A.corner_rows || A.corner_cols) {
    throw Fail{PSG_E_CORNER_FORBIDDEN, "corner block not allowed for this kind"};
  }
  const size_t want = body_entry_count(A.kind, n, m, s, r);
  if (A.data_len != want)
    throw Fail{PSG_E_DIMENSION_MISMATCH,
               "expected " + std::to_string(want) + " body entries, got " + std::to_string(A.data_len)};
}

// ----------------------------------------------------------------------------
// partition plan: plan_partition (src/partition.cpp:52-105), kept in closed
// form (no O(p) host arrays on the factor path).
// ----------------------------------------------------------------------------
struct Plan {
  int kind = 0, n = 0, m = 1, p = 0, sep_size = 0;
  bool has_corner = false;
  int unit = 1, k_units = 1;
  long base = 0, rem = 0;
  int sep_count() const { return has_corner ? p + 1 : p - 1; }
  long body_begin_units(int i) const {
    return (has_corner ? k_units : 0) + (long)i * base + std::min<long>(i, rem) + (long)i * k_units;
  }
  int body_begin(int i) const { return int(body_begin_units(i) * unit); }
  int body_end(int i) const { return int((body_begin_units(i) + base + (i < rem ? 1 : 0)) * unit); }
  int sep_start(int j) const {
    if (has_corner) return j == 0 ? 0 : body_end(j - 1);
    return body_end(j);
  }
};

Plan make_plan(const psg_desc& A, int p) {
  if (p < 2) throw Fail{PSG_E_TOO_MANY_PARTITIONS, "p must be >= 2"};
  if (A.kind == PSG_CIRCULANT && A.r != 0)  // src/partition.cpp:53-55
    throw Fail{PSG_E_UNSUPPORTED_KIND, "circulant-like corner content is not canonical; permute_corner first"};
  Plan P;
  P.kind = A.kind;
  P.n = A.n;
  P.m = A.m;
  P.p = p;
  const bool scalar = A.kind == PSG_BANDED || A.kind == PSG_CIRCULANT;
  P.sep_size = scalar ? std::max(A.s, A.r) : A.m;
  P.has_corner = A.kind == PSG_BABD || A.kind == PSG_CIRCULANT;
  const int k = P.sep_size;
  const long seps = P.has_corner ? p + 1L : p - 1L;
  P.unit = scalar ? 1 : A.m;
  if (k % P.unit != 0) throw Fail{PSG_E_UNSUPPORTED_KIND, "separator does not tile blocks"};
  const long n_units = A.n / P.unit;
  P.k_units = k / P.unit;
  const long body_total = n_units - seps * P.k_units;
  const long min_body = std::max(1, P.k_units);
  if (body_total < (long)p * min_body)
    throw Fail{PSG_E_TOO_MANY_PARTITIONS, "n too small for p = " + std::to_string(p) + " partitions of this kind"};
  P.base = body_total / p;
  P.rem = body_total % p;
  return P;
}

// ----------------------------------------------------------------------------
// small pools: CUDA events
// ----------------------------------------------------------------------------
struct EventPool {
  // events belong to the device that was current when they were created:
  // the free lists are kept per device (a handle releases its events while
  // its own device is current, psg_release's DeviceGuard)
  std::mutex mu;
  std::map<int, std::vector<cudaEvent_t>> free_;
  cudaEvent_t get() {
    const int dev = BlockCache::device();
    {
      std::lock_guard<std::mutex> g(mu);
      auto& fl = free_[dev];
      if (!fl.empty()) {
        cudaEvent_t e = fl.back();
        fl.pop_back();
        return e;
      }
    }
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    return e;
  }
  void put(cudaEvent_t e) {
    const int dev = BlockCache::device();
    std::lock_guard<std::mutex> g(mu);
    free_[dev].push_back(e);
  }
};

EventPool& event_pool() {
  static EventPool* p = new EventPool;
  return *p;
}

// Process-wide copy streams per device (host-buffer pipelines): one for each
// PCIe direction, non-blocking, ordered against the compute stream by events.
void copy_streams(cudaStream_t& in, cudaStream_t& out) {
  static std::mutex mu;
  static std::map<int, std::pair<cudaStream_t, cudaStream_t>> by_dev;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  auto it = by_dev.find(dev);
  if (it == by_dev.end()) {
    cudaStream_t a, b;
    CUDA_TRY(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
    it = by_dev.emplace(dev, std::make_pair(a, b)).first;
  }
  in = it->second.first;
  out = it->second.second;
}

// ----------------------------------------------------------------------------
// Tridiagonal solver: speculative single-level path + exact multi-level path
// ----------------------------------------------------------------------------
constexpr int kMaxSeg = 32 * 33;  // 1056 rows per segment (one warp)
constexpr int kMinSpecSeg = 2 * kHalo + 1;

struct TriLevel {
  TriRows A{};
  RowArr F{};
  double* x = nullptr;  // output of this level (rows of this level's system)
  int q = 0;            // rows
  SegMap S{};
  int maxlen = 0;
  DevBuf<int> start, len;                              // refined maps only
  DevBuf<double> mat, rhsv;                            // 4*nseg, 2*nseg
  DevBuf<double> Tsub, Tdiag, Tsup, rhs_next, x_next;  // nseg-1
};

// q rows -> segments of <= kMaxSeg rows separated by single rows, using the
// reference plan formula (equal bodies, remainder to the leading ones).
SegMap segment_uniform(int q, int& maxlen) {
  if (q <= kMaxSeg) {
    maxlen = q;
    return SegMap{1, q, 0, nullptr, nullptr};
  }
  const int p = (q + 1 + 1023) / 1024;  // ~1023-row bodies
  const long body_total = (long)q - (p - 1);
  const int base = int(body_total / p), rem = int(body_total % p);
  maxlen = base + (rem ? 1 : 0);
  return SegMap{p, base, rem, nullptr, nullptr};
}

template <int M, bool BODY>
void launch_segment_solve_t(const TriSolveArgs& a, int nseg, cudaStream_t s, bool pdl) {
  constexpr int bytes = TriWarpSmem<M>::BYTES;
  if (pdl)
    launch_pdl(tri_segment_solve_kernel<M, false, BODY>, dim3(nseg), dim3(32), bytes, s, a);
  else
    tri_segment_solve_kernel<M, false, BODY><<<nseg, 32, bytes, s>>>(a);
}

template <int M>
void launch_segment_solve(const TriSolveArgs& a, int nseg, cudaStream_t s, bool pdl) {
  if (a.body)
    launch_segment_solve_t<M, true>(a, nseg, s, pdl);
  else
    launch_segment_solve_t<M, false>(a, nseg, s, pdl);
}

// pdl: K3 stages A and F before waiting for its predecessor -- only valid
// when neither is produced by the preceding kernel (the speculative solve:
// user f, predecessor = the separator kernel)
int sm_count() {
  static int n = [] {
    int dev = 0, c = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    return c > 0 ? c : 148;
  }();
  return n;
}

// persistent K3 (two staging buffers per warp) for 33-row chunks: segments
// [a.seg0, a.seg0 + nseg) by sm_count() * per-SM warps
void launch_segment_solve_persist(TriSolveArgs a, int nseg, cudaStream_t s, bool pdl) {
  constexpr int bytes = 2 * TriWarpSmem<33>::BYTES;
  ensure_smem(reinterpret_cast<const void*>(tri_segment_solve_kernel<33, true>), bytes);
  static const int per_sm = [] {
    const char* e = getenv("PSG_K3_PERSIST");
    return e && atoi(e) > 0 ? atoi(e) : 3;
  }();
  const int grid = std::min(nseg, sm_count() * per_sm);
  a.seg_end = a.seg0 + nseg;
  if (pdl)
    launch_pdl(tri_segment_solve_kernel<33, true>, dim3(grid), dim3(32), bytes, s, a);
  else
    tri_segment_solve_kernel<33, true><<<grid, 32, bytes, s>>>(a);
}

void segment_solve(const TriSolveArgs& a, int nseg, int maxlen, cudaStream_t s, bool pdl = false,
                   bool persist = false) {
  // off unless PSG_K3_PERSIST = warps per SM is set: measured slower (3 warps
  // per SM: 0.558 ms/step against 0.451 for one warp per segment)
  static const bool persist_on = [] {
    const char* e = getenv("PSG_K3_PERSIST");
    return e && atoi(e) > 0;
  }();
  if (persist && persist_on && !a.body && maxlen > 32 * 17 && maxlen <= 32 * 33 && nseg > 4 * sm_count()) {
    launch_segment_solve_persist(a, nseg, s, pdl);
    LAUNCH_CHECK();
    return;
  }
  if (maxlen <= 32 * 5)
    launch_segment_solve<5>(a, nseg, s, pdl);
  else if (maxlen <= 32 * 9)
    launch_segment_solve<9>(a, nseg, s, pdl);
  else if (maxlen <= 32 * 17)
    launch_segment_solve<17>(a, nseg, s, pdl);
  else if (maxlen <= 32 * 33)
    launch_segment_solve<33>(a, nseg, s, pdl);
  else
    throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "segment longer than the per-warp capacity"};
  LAUNCH_CHECK();
}

int blocks_for(long work, int tpb) { return (int)((work + tpb - 1) / tpb); }

struct TriSolver {
  // level-0 system
  TriRows A0{};
  int n = 0;
  SegMap S0{};
  int maxlen0 = 0, minlen0 = 0;
  DevBuf<int> start0, len0;  // refined maps
  // speculative path buffers
  DevBuf<double> Tdiag, xsep, xsep_alt;  // two separator buffers: consecutive solves alternate (see spec_solve)
  DevBuf<double4> crec;  // per-segment certificate records
  DevBuf<unsigned> cctr;  // certificate kernel: finished-block counter (last block publishes the status)
  bool body_cert = false; // K3 also certifies every body row (PSG_OPT_BODY_CERT)
  // exact multi-level path (built on demand)
  std::vector<std::unique_ptr<TriLevel>> lv;
  int launches = 0;

  void init(const TriRows& A, int n_, const SegMap& S, int maxlen, int minlen, const std::vector<int>* st,
            const std::vector<int>* ln, cudaStream_t s) {
    A0 = A;
    n = n_;
    S0 = S;
    maxlen0 = maxlen;
    minlen0 = minlen;
    hstart0.clear();
    if (st) hstart0 = *st;
    if (st) {
      start0.alloc(st->size());
      len0.alloc(ln->size());
      CUDA_TRY(cudaMemcpyAsync(start0.p, st->data(), sizeof(int) * st->size(), cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(len0.p, ln->data(), sizeof(int) * ln->size(), cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaStreamSynchronize(s));  // pageable source
      S0.start = start0.p;
      S0.len = len0.p;
    }
    crec.alloc(S0.nseg);
    cctr.alloc(1);
    CUDA_TRY(cudaMemsetAsync(cctr.p, 0, sizeof(unsigned), s));
    if (S0.nseg > 1) {
      xsep.alloc(S0.nseg - 1);
      xsep_alt.alloc(S0.nseg - 1);
    }
  }

  bool spec_possible() const { return minlen0 >= kMinSpecSeg && S0.nseg > 1; }

  // ---- speculative path ----------------------------------------------------
  // The speculative factor is lazy: its sweeps run inside the next solve's
  // separator kernel (tri_spec_fused_kernel, one pass over the windows of
  // a, b, c and f).  tdiag_current: Tdiag matches the current matrix.
  bool tdiag_current = false;
  void spec_factor(cudaStream_t) {
    Tdiag.alloc(S0.nseg - 1);
    tdiag_current = false;
  }
  // the factor alone (Tdiag for psg_reduced_blocks, no solve)
  void spec_tdiag(cudaStream_t s) {
    if (tdiag_current) return;
    const int nsep = S0.nseg - 1;
    tri_spec_fused_kernel<false><<<blocks_for(nsep, kFacSeps), 32, 0, s>>>(A0, RowArr{}, S0, nullptr, Tdiag.p,
                                                                          nullptr, 0, nsep);
    LAUNCH_CHECK();
    launches += 1;
    tdiag_current = true;
  }
  // pdl: may overlap the previous solve's certificate kernel (see the kernel)
  void fused_sep(const RowArr& F, DevStatus* st, int ja, int jb, cudaStream_t s, bool pdl = false) {
    const dim3 grid(std::max(1, blocks_for(jb - ja, kFacSeps)));
    if (pdl)
      launch_pdl(tri_spec_fused_kernel<true>, grid, dim3(32), 0, s, A0, F, S0, xsep.p, Tdiag.p, st, ja, jb);
    else
      tri_spec_fused_kernel<true><<<grid, 32, 0, s>>>(A0, F, S0, xsep.p, Tdiag.p, st, ja, jb);
    LAUNCH_CHECK();
    launches += 1;
  }

  // level-0 back-substitution and separator certificate
  // host_out: a pinned host slot the certificate kernel publishes the final status to
  void k3_and_cert(const RowArr& F, double* x, const double* xs, DevStatus* st, cudaStream_t s, bool pdl = false,
                   DevStatus* host_out = nullptr) {
    TriSolveArgs a{};
    a.A = A0;
    a.F = F;
    a.S = S0;
    a.xsep = xs;
    a.x = x;
    a.crec = crec.p;
    a.status = st;
    a.body = body_cert ? 1 : 0;
    // the separator certificate stays a separate PDL-chained kernel: folding it
    // into K3 (each segment's arrival at its two separators, the later one
    // evaluating omega, the last segment publishing the status) held every K3
    // warp for its fences and atomics -- config 1 0.455 -> 0.694 ms/step
    //
    segment_solve(a, S0.nseg, maxlen0, s, pdl, /*persist=*/true);
    launch_pdl(tri_cert_kernel, dim3(blocks_for(S0.nseg - 1, 256)), dim3(256), 0, s, S0.nseg - 1,
               (const double4*)crec.p, st, host_out, cctr.p);
    launches += 2;
  }

  void spec_solve(const RowArr& F, double* x, DevStatus* st, cudaStream_t s, cudaEvent_t* ev,
                  DevStatus* host_out = nullptr) {
    const int nsep = S0.nseg - 1;
    // consecutive solves alternate separator buffers: the next solve's
    // separator kernel may run while this solve's K3 drains (K3 and the
    // certificate kernel trigger their dependents early; the separator kernel
    // completes only after the previous certificate, so the next K3 -- which
    // waits on it -- never overlaps this one's writes)
    std::swap(xsep.p, xsep_alt.p);
    fused_sep(F, st, 0, nsep, s, /*pdl=*/true);  // factor sweeps + separator values in one pass
    tdiag_current = true;
    if (ev) {  // the speculative reduced matrix is diagonal: phase 2 is fused into phase 1
      CUDA_TRY(cudaEventRecord(ev[1], s));
      CUDA_TRY(cudaEventRecord(ev[2], s));
    }
    k3_and_cert(F, x, xsep.p, st, s, /*pdl=*/true, host_out);  // K3 stages its rows while the separators finish
  }

  // ---- host buffers: chunked pipeline ---------------------------------------
  // f arrives in row chunks on copy stream `ci`; the separators whose windows
  // are complete and the segments between them are solved per chunk on `s`;
  // each chunk of x leaves on copy stream `co` while later chunks of f are
  // still arriving (both PCIe directions busy at once).  Same kernels and
  // arithmetic as spec_solve; the certificate covers every separator.
  void spec_solve_host(const double* hf, double* hx, double* df, double* dx, DevStatus* st, cudaStream_t s,
                       cudaStream_t ci, cudaStream_t co, cudaEvent_t* evs, int nchunk, DevStatus* host_out) {
    const int nsep = S0.nseg - 1;
    auto seg_start = [&](int i) -> long {  // first row of segment i (n for i == nseg)
      if (i >= S0.nseg) return n;
      if (S0.start) return hstart0[i];
      return (long)i * (S0.base + 1) + (i < S0.rem ? i : S0.rem);
    };
    // entry: the previous users of df / dx on s are done before the copies
    CUDA_TRY(cudaEventRecord(evs[0], s));
    CUDA_TRY(cudaStreamWaitEvent(ci, evs[0], 0));
    CUDA_TRY(cudaStreamWaitEvent(co, evs[0], 0));
    const RowArr F = make_rows(df, 0, n);
    int ja = 0;  // separators done
    for (int g = 0; g < nchunk; ++g) {
      const long r0 = (long)n * g / nchunk, r1 = (long)n * (g + 1) / nchunk;
      CUDA_TRY(cudaMemcpyAsync(df + r0, hf + r0, sizeof(double) * (r1 - r0), cudaMemcpyHostToDevice, ci));
      CUDA_TRY(cudaEventRecord(evs[1 + 2 * g], ci));
      CUDA_TRY(cudaStreamWaitEvent(s, evs[1 + 2 * g], 0));
      // separators whose f window (t +- 32) lies in rows < r1; all of them at the end
      int jb = ja;
      if (g == nchunk - 1) {
        jb = nsep;
      } else {
        while (jb < nsep && seg_start(jb + 1) - 1 + kHalo < r1) ++jb;
      }
      const int ib = g == nchunk - 1 ? S0.nseg : jb;  // segments with both separators known
      const int ia = ja == 0 ? 0 : ja;
      if (jb > ja || g == 0) fused_sep(F, g == 0 ? st : nullptr, ja, jb, s);  // chunk 0 also resets the status
      if (ib > ia) {
        TriSolveArgs a{};
        a.A = A0;
        a.F = F;
        a.S = S0;
        a.xsep = xsep.p;
        a.x = dx;
        a.crec = crec.p;
        a.status = st;
        a.seg0 = ia;
        a.body = body_cert ? 1 : 0;
        segment_solve(a, ib - ia, maxlen0, s, /*pdl=*/true);
        launches += 1;
        CUDA_TRY(cudaEventRecord(evs[2 + 2 * g], s));
        CUDA_TRY(cudaStreamWaitEvent(co, evs[2 + 2 * g], 0));
        const long x0 = seg_start(ia), x1 = seg_start(ib);
        CUDA_TRY(cudaMemcpyAsync(hx + x0, dx + x0, sizeof(double) * (x1 - x0), cudaMemcpyDeviceToHost, co));
      }
      ja = jb;
    }
    launch_pdl(tri_cert_kernel, dim3(blocks_for(nsep, 256)), dim3(256), 0, s, nsep, (const double4*)crec.p, st,
               host_out, cctr.p);
    launches += 1;
    tdiag_current = true;
    CUDA_TRY(cudaEventRecord(evs[0], co));
    CUDA_TRY(cudaStreamWaitEvent(s, evs[0], 0));  // x is on the host when s reaches this point
  }
  std::vector<int> hstart0;  // host copy of S0's explicit starts (refined maps)

  // ---- exact multi-level path ----------------------------------------------
  void build_levels(cudaStream_t s) {
    if (!lv.empty()) return;
    auto L0 = std::make_unique<TriLevel>();
    L0->A = A0;
    L0->q = n;
    L0->S = S0;
    L0->maxlen = maxlen0;
    lv.push_back(std::move(L0));
    for (;;) {
      TriLevel& L = *lv.back();
      const int nseg = L.S.nseg;
      if (nseg == 1) break;
      const int ns = nseg - 1;
      L.mat.alloc(4 * (size_t)nseg);
      L.rhsv.alloc(2 * (size_t)nseg);
      L.Tsub.alloc(ns);
      L.Tdiag.alloc(ns);
      L.Tsup.alloc(ns);
      L.rhs_next.alloc(ns);
      L.x_next.alloc(ns);
      auto N = std::make_unique<TriLevel>();
      N->A.a = make_rows(L.Tsub.p, 1, ns);
      N->A.b = make_rows(L.Tdiag.p, 0, ns);
      N->A.c = make_rows(L.Tsup.p, 0, ns - 1);
      N->F = make_rows(L.rhs_next.p, 0, ns);
      N->x = L.x_next.p;
      N->q = ns;
      N->S = segment_uniform(ns, N->maxlen);
      lv.push_back(std::move(N));
    }
    (void)s;
  }

  void exact_factor(cudaStream_t s) {
    build_levels(s);
    for (size_t l = 0; l + 1 < lv.size(); ++l) {
      TriLevel& L = *lv[l];
      tri_interface_kernel<true, false><<<blocks_for(2L * L.S.nseg, 128), 128, 0, s>>>(
          L.A, make_rows(nullptr, 0, 0), L.S, 0, L.mat.p, nullptr);
      LAUNCH_CHECK();
      tri_assemble_matrix_kernel<<<blocks_for(L.S.nseg - 1, 256), 256, 0, s>>>(L.A, L.S, L.mat.p, L.Tsub.p,
                                                                               L.Tdiag.p, L.Tsup.p);
      LAUNCH_CHECK();
      launches += 2;
    }
  }

  // Exact solve of level `from` (0 = the user system, 1 = the reduced system).
  void exact_solve(const RowArr& F0, double* x0, DevStatus* st, cudaStream_t s, cudaEvent_t* ev, size_t from = 0) {
    lv[from]->F = F0;
    lv[from]->x = x0;
    for (size_t l = from; l + 1 < lv.size(); ++l) {
      TriLevel& L = *lv[l];
      tri_interface_kernel<false, true><<<blocks_for(2L * L.S.nseg, 128), 128, 0, s>>>(L.A, L.F, L.S, 0, nullptr,
                                                                                      L.rhsv.p);
      LAUNCH_CHECK();
      tri_assemble_rhs_kernel<<<blocks_for(L.S.nseg - 1, 256), 256, 0, s>>>(L.A, L.F, L.S, L.rhsv.p, L.rhs_next.p);
      LAUNCH_CHECK();
      launches += 2;
      if (l == from && ev) CUDA_TRY(cudaEventRecord(ev[1], s));
    }
    for (size_t l = lv.size(); l-- > from;) {
      TriLevel& L = *lv[l];
      if (l == from && ev) CUDA_TRY(cudaEventRecord(ev[2], s));
      if (l == 0 && L.S.nseg > 1 && st) {
        k3_and_cert(L.F, L.x, L.x_next.p, st, s);
        continue;
      }
      TriSolveArgs a{};
      a.A = L.A;
      a.F = L.F;
      a.S = L.S;
      a.xsep = L.S.nseg > 1 ? L.x_next.p : nullptr;
      a.x = L.x;
      a.status = l == 0 ? st : nullptr;  // pivots/non-finite values are attributed at level 0 only
      segment_solve(a, L.S.nseg, L.maxlen, s);
      launches += 1;
    }
  }

  void restore_level1_wiring() {
    if (lv.size() > 1) {
      lv[1]->x = lv[0]->x_next.p;
      lv[1]->F = make_rows(lv[0]->rhs_next.p, 0, lv[1]->q);
    }
  }

  // phase 1 of the exact path alone: the level-0 reduced right-hand side
  // (f at the separators plus every body's condensed contribution) lands in
  // lv[0]->rhs_next
  const double* exact_condense(const RowArr& F0, cudaStream_t s) {
    TriLevel& L = *lv[0];
    L.F = F0;
    tri_interface_kernel<false, true><<<blocks_for(2L * L.S.nseg, 128), 128, 0, s>>>(L.A, L.F, L.S, 0, nullptr,
                                                                                    L.rhsv.p);
    LAUNCH_CHECK();
    tri_assemble_rhs_kernel<<<blocks_for(L.S.nseg - 1, 256), 256, 0, s>>>(L.A, L.F, L.S, L.rhsv.p, L.rhs_next.p);
    LAUNCH_CHECK();
    return L.rhs_next.p;
  }

};

// ----------------------------------------------------------------------------
// Generic exact solver (every kind): multi-level partition method over
// structured views; the reduced matrix of each level is the next level's
// StructuredMatrix (block tridiagonal, or ABD row layout + corner).
// ----------------------------------------------------------------------------
void envelope_of(int kind, int m, int s, int r, int& es, int& er) {  // scalar_envelope
  if (kind == PSG_BANDED) {
    es = s;
    er = r;
  } else if (kind == PSG_BLOCKTRI) {
    es = er = 2 * m - 1;
  } else {
    es = m - 1 + s;
    er = m - 1 + r;
  }
}

// ----------------------------------------------------------------------------
// K x K block speculative path (blk_kernels.cuh)
// ----------------------------------------------------------------------------
// banded band bases: A(row, row + d) = data[boff[d + K] + row] (structmat.cpp:33-38 layout)
void fill_band_offsets(BlkArgs& a, int K, long n, int s_, int r_, size_t data_len) {
  for (int t = 0; t < 9; ++t) a.boff[t] = 0;
  long off = 0;
  for (int d = -s_; d <= r_; ++d) {
    if (d + K >= 0 && d + K < 9) a.boff[d + K] = off - (d < 0 ? -d : 0);
    off += n - (d < 0 ? -d : d);
  }
  a.data_len = (long)data_len;
}

template <int K, int M, int LAYOUT, int NW>
void launch_blk_kernel(const BlkArgs& a, cudaStream_t s, bool pdl) {
  constexpr int bytes = BlkSmem<K, M, NW>::bytes(LAYOUT);
  ensure_smem(reinterpret_cast<const void*>(blk_segment_solve_kernel<K, M, LAYOUT, NW>), bytes);
  if (pdl)
    launch_pdl(blk_segment_solve_kernel<K, M, LAYOUT, NW>, dim3(a.nseg), dim3(32 * NW), bytes, s, a);
  else
    blk_segment_solve_kernel<K, M, LAYOUT, NW><<<a.nseg, 32 * NW, bytes, s>>>(a);
  LAUNCH_CHECK();
}

// chunk depth M and warps NW per body: 32 NW M block rows per body
struct BlkShape {
  int M, NW;
};
BlkShape blk_shape(int K, int NB) {
  if (K == 4) return NB <= 64 ? BlkShape{2, 1} : (NB <= 128 ? BlkShape{2, 2} : BlkShape{0, 0});
  if (K == 3)
    return NB <= 64 ? BlkShape{2, 1} : (NB <= 96 ? BlkShape{3, 1} : (NB <= 192 ? BlkShape{3, 2} : BlkShape{0, 0}));
  if (K == 2)
    return NB <= 96 ? BlkShape{3, 1} : (NB <= 160 ? BlkShape{5, 1} : (NB <= 320 ? BlkShape{5, 2} : BlkShape{0, 0}));
  return BlkShape{0, 0};
}
int blk_max_nb(int K) { return K == 4 ? 128 : (K == 3 ? 192 : 320); }

template <int K, int MC, int LPB>
void launch_blk_narrow(const BlkArgs& a, cudaStream_t s, bool pdl) {
  constexpr int bytes = BlkNarrow<K, MC, LPB>::BYTES;
  ensure_smem(reinterpret_cast<const void*>(blk_body_narrow_kernel<K, MC, LPB>), bytes);
  constexpr int G = 32 / LPB;
  if (pdl)
    launch_pdl(blk_body_narrow_kernel<K, MC, LPB>, dim3((a.nseg + G - 1) / G), dim3(32), bytes, s, a);
  else
    blk_body_narrow_kernel<K, MC, LPB><<<(a.nseg + G - 1) / G, 32, bytes, s>>>(a);
  LAUNCH_CHECK();
}


// pdl: the body kernel stages A and f before waiting for its predecessor --
// only for the speculative solve (user f, predecessor = the separator kernel)
bool launch_blk_segments(int K, int NB, int layout, const BlkArgs& a, cudaStream_t s, bool pdl = false) {
  if (layout == kBlkBlockTri && K == 4) {  // narrow body kernel: 4 block rows per lane, 16 or 32 lanes per body
    if (NB <= 64) return launch_blk_narrow<4, 4, 16>(a, s, pdl), true;
    if (NB <= 128) return launch_blk_narrow<4, 4, 32>(a, s, pdl), true;
  }
  const BlkShape sh = blk_shape(K, NB);
#define PSG_BLK_CASE(KK_, MM_, NW_)                                              \
  if (K == KK_ && sh.M == MM_ && sh.NW == NW_) {                                 \
    if (layout == kBlkBlockTri)                                                  \
      launch_blk_kernel<KK_, MM_, kBlkBlockTri, NW_>(a, s, pdl);                 \
    else                                                                         \
      launch_blk_kernel<KK_, MM_, kBlkBanded, NW_>(a, s, pdl);                   \
    return true;                                                                 \
  }
  PSG_BLK_CASE(4, 2, 1)
  PSG_BLK_CASE(4, 2, 2)
  PSG_BLK_CASE(3, 2, 1)
  PSG_BLK_CASE(3, 3, 1)
  PSG_BLK_CASE(3, 3, 2)
  PSG_BLK_CASE(2, 3, 1)
  PSG_BLK_CASE(2, 5, 1)
  PSG_BLK_CASE(2, 5, 2)
#undef PSG_BLK_CASE
  return false;
}

// truncation depth in block rows per side (about 64 scalar rows)
constexpr int blk_hb(int K) { return K == 2 ? 32 : 16; }

// Banded s, r <= K in scalar band arithmetic (band_kernels.cuh): longest
// body of one body kernel (rows; smem (2K + 2) x (L + 4) doubles per warp).
// PSG_BAND_OLD=1 keeps the K x K block kernels for banded matrices.
int band_max_rows() {
  static const int v = [] {
    const char* e = getenv("PSG_BAND_MAXL");
    return e && atoi(e) > 0 ? atoi(e) : 576;
  }();
  return v;
}
// Block tridiagonal bodies: two threads per body (blktri_body_kernel) unless
// PSG_BLK_BODY_NARROW=1 (the warp-per-body lane-chunk kernels).
bool blktri_thread_bodies() {
  static const bool v = [] {
    const char* e = getenv("PSG_BLK_BODY_NARROW");
    return !(e && atoi(e) > 0);
  }();
  return v;
}
bool band_scalar_enabled() {
  static const bool v = [] {
    const char* e = getenv("PSG_BAND_OLD");
    return !(e && atoi(e) > 0);
  }();
  return v;
}

// Speculative solver for the K x K block kinds.  Its bodies are the
// reference plan's, each split into equal sub-bodies (extra K-row separators)
// when longer than one warp's 32 M block rows.
struct BlkSolver {
  int K = 0, layout = 0, NB = 0;
  bool band = false;  // scalar band kernels (band_kernels.cuh)
  bool tbody = false; // block tridiagonal: two threads per body (blktri_body_kernel)
  int RB = 0;         // band: smem rows per array
  DevBuf<double> scr; // tbody: the bodies' parked (G, z) records, (K^2 + K) per block row
  bool possible = false;
  BlkArgs base{};
  std::vector<GPart> hpart;
  std::vector<int> hsep;
  DevBuf<GPart> part;
  DevBuf<int> sep;
  DevBuf<double> Tdiag, xsep, rec;
  DevBuf<unsigned> cctr;  // certificate kernel: finished-block counter (last block publishes the status)
  int nseg = 0, nsep = 0, launches = 0;

  void init(const psg_desc& A, const Plan& P) {
    possible = false;
    if (P.has_corner) return;
    if (A.kind == PSG_BLOCKTRI && A.m >= 2 && A.m <= 4) {
      K = A.m;
      layout = kBlkBlockTri;
    } else if (A.kind == PSG_BANDED && P.sep_size >= 2 && P.sep_size <= 4) {
      K = P.sep_size;
      layout = kBlkBanded;
    } else {
      return;
    }
    const int unit = layout == kBlkBlockTri ? K : 1, ku = K / unit;
    band = layout == kBlkBanded && band_scalar_enabled();
    tbody = layout == kBlkBlockTri && blktri_thread_bodies();
    // longest body of one kernel, in block rows of K (two-thread bodies: the
    // reference plan's own bodies, not merged -- twice the threads in flight)
    const int maxnb = band ? band_max_rows() / K : (tbody ? INT_MAX : blk_max_nb(K));
    const int mergenb = tbody ? 0 : maxnb;
    hpart.clear();
    hsep.clear();
    int maxL = 0, minL = INT_MAX;
    // reference bodies, neighbours merged (with the separator between them)
    // while the union still fits one body kernel: fewer separators means less
    // factor / separator work for the same body work
    std::vector<std::pair<int, int>> bodies;
    for (int i = 0; i < P.p; ++i) {
      const int b = P.body_begin(i), L = P.body_end(i) - b;
      if (!bodies.empty()) {
        auto& c = bodies.back();
        const int merged = c.second + K + L;
        if ((merged + K - 1) / K <= mergenb) {
          c.second = merged;
          continue;
        }
      }
      bodies.emplace_back(b, L);
    }
    for (size_t i = 0; i < bodies.size(); ++i) {
      const int b = bodies[i].first, L = bodies[i].second;
      const int Lu = L / unit;
      auto nb_of = [&](int t) { return (((Lu - (t - 1) * ku) + t - 1) / t * unit + K - 1) / K; };
      int t = 1;
      while (t < Lu && nb_of(t) > maxnb) ++t;
      const int body = Lu - (t - 1) * ku, bs = body / t, br = body % t;
      int cur = b;
      for (int u = 0; u < t; ++u) {
        const int len = (bs + (u < br ? 1 : 0)) * unit;
        hpart.push_back(GPart{cur, len, -1, -1});
        maxL = std::max(maxL, len);
        minL = std::min(minL, len);
        cur += len;
        if (u + 1 < t || i + 1 < bodies.size()) {
          hsep.push_back(cur);
          cur += K;
        }
      }
    }
    nseg = (int)hpart.size();
    nsep = (int)hsep.size();
    for (int g = 0; g < nseg; ++g) {
      hpart[g].ls = g > 0 ? hsep[g - 1] : -1;
      hpart[g].rs = g < nsep ? hsep[g] : -1;
    }
    NB = (maxL + K - 1) / K;
    if (minL < blk_hb(K) * K || minL < 2 * K || nsep < 1) return;
    if (band) {
      if (minL < 4 * K || maxL > band_max_rows()) return;
      RB = (maxL + 4) & ~1;
    } else if (tbody) {
      if (minL < 2 * K) return;
      scr.alloc((size_t)(A.n / K) * (K * K + K) + 8);
    } else if (blk_shape(K, NB).M == 0) {
      return;
    }
    part.alloc(nseg);
    sep.alloc(nsep);
    CUDA_TRY(cudaMemcpy(part.p, hpart.data(), sizeof(GPart) * nseg, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(sep.p, hsep.data(), sizeof(int) * nsep, cudaMemcpyHostToDevice));
    Tdiag.alloc((size_t)nsep * K * K);
    xsep.alloc((size_t)nsep * K);
    rec.alloc((size_t)nseg * 4 * K);
    cctr.alloc(1);
    CUDA_TRY(cudaMemset(cctr.p, 0, sizeof(unsigned)));
    base.n = A.n;
    base.s = A.s;
    base.r = A.r;
    base.data = A.data;
    base.part = part.p;
    base.nseg = nseg;
    fill_band_offsets(base, K, A.n, A.s, A.r, A.data_len);
    possible = true;
  }

  void set_data(const double* d) { base.data = d; }

  template <int KK>
  void band_spec_launch_k(const BlkSpecArgs& g, cudaStream_t s) {
    constexpr int W = blk_hb(KK) * KK;
    const int grid = (nsep + 31) / 32;
    band_spec_kernel<KK, W><<<grid, kBandSpecThreads, 0, s>>>(g);
  }
  void band_spec_launch(const BlkSpecArgs& g, cudaStream_t s) {
    if (K == 4)
      band_spec_launch_k<4>(g, s);
    else if (K == 3)
      band_spec_launch_k<3>(g, s);
    else
      band_spec_launch_k<2>(g, s);
  }
  template <int KK>
  void band_body_launch_k(const BlkArgs& a, cudaStream_t s) {
    const int bytes = 8 * (2 * KK + 2) * RB;
    ensure_smem(reinterpret_cast<const void*>(band_body_kernel<KK>), 200 * 1024);
    launch_pdl(band_body_kernel<KK>, dim3(a.nseg), dim3(32), bytes, s, a, RB);
  }
  void band_body_launch(const BlkArgs& a, cudaStream_t s) {
    if (K == 4)
      band_body_launch_k<4>(a, s);
    else if (K == 3)
      band_body_launch_k<3>(a, s);
    else
      band_body_launch_k<2>(a, s);
    LAUNCH_CHECK();
  }

  // the factor is lazy: its block sweeps run inside the next solve's fused
  // separator kernel (blk_spec_fused_kernel), which also condenses f
  void spec_factor(cudaStream_t) {}

  // fused factor + separators -> bodies -> certificate; the first kernel resets the status slot.
  void spec_solve(const double* f, double* x, DevStatus* st, cudaStream_t s, cudaEvent_t* ev,
                  DevStatus* host_out = nullptr) {
    BlkSpecArgs g{};
    g.data = base.data;
    g.n = base.n;
    g.s = base.s;
    g.r = base.r;
    g.layout = layout;
    g.nsep = nsep;
    g.sep = sep.p;
    g.f = f;
    g.xsep = xsep.p;
    g.Tdiag = Tdiag.p;
    g.reset = st;
    for (int t = 0; t < 9; ++t) g.boff[t] = base.boff[t];
    g.data_len = base.data_len;
    constexpr int NS = 1;  // separators per warp (2, chains interleaved: config 2 82 -> 123 us, config 3 217 -> 332 us)
    const int grid = (nsep + 4 * NS - 1) / (4 * NS);
    static const bool warp_spec = [] {  // PSG_BLK_SPEC_WARP=1: the round-1/2 warp-per-separator kernel
      const char* e = getenv("PSG_BLK_SPEC_WARP");
      return e && atoi(e) > 0;
    }();
    if (band) {
      band_spec_launch(g, s);
    } else if (!warp_spec) {
      const int g2 = (nsep + 31) / 32;
      if (K == 4)
        blktri_spec_kernel<4, blk_hb(4)><<<g2, 64, 0, s>>>(g);
      else if (K == 3)
        blktri_spec_kernel<3, blk_hb(3)><<<g2, 64, 0, s>>>(g);
      else
        blktri_spec_kernel<2, blk_hb(2)><<<g2, 64, 0, s>>>(g);
    } else if (K == 4)
      blk_spec_fused_kernel<4, blk_hb(4), NS><<<grid, 128, 0, s>>>(g);
    else if (K == 3)
      blk_spec_fused_kernel<3, blk_hb(3), NS><<<grid, 128, 0, s>>>(g);
    else
      blk_spec_fused_kernel<2, blk_hb(2), NS><<<grid, 128, 0, s>>>(g);
    LAUNCH_CHECK();
    if (ev) {
      CUDA_TRY(cudaEventRecord(ev[1], s));
      CUDA_TRY(cudaEventRecord(ev[2], s));
    }
    BlkArgs a = base;
    a.f = f;
    a.x = x;
    a.xsep = xsep.p;
    a.rec = rec.p;
    a.status = st;
    if (band) {
      band_body_launch(a, s);
    } else if (tbody) {
      const dim3 grid((nseg + 31) / 32);
      if (K == 4)
        launch_pdl(blktri_body_kernel<4>, grid, dim3(64), 0, s, a, scr.p);
      else if (K == 3)
        launch_pdl(blktri_body_kernel<3>, grid, dim3(64), 0, s, a, scr.p);
      else
        launch_pdl(blktri_body_kernel<2>, grid, dim3(64), 0, s, a, scr.p);
      LAUNCH_CHECK();
    } else if (!launch_blk_segments(K, NB, layout, a, s, /*pdl=*/true))
      throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "block body too long"};
    const int cg = std::min(148 * 8, (nsep * K + 255) / 256);
    const double* Td = Tdiag.p;
    const int* sp = sep.p;
    const double* xs = xsep.p;
    const double* rc = rec.p;
    unsigned* dc = cctr.p;
    if (K == 4)
      launch_pdl(blk_cert_kernel<4>, dim3(cg), dim3(256), 0, s, Td, sp, nsep, f, xs, rc, st, host_out, dc);
    else if (K == 3)
      launch_pdl(blk_cert_kernel<3>, dim3(cg), dim3(256), 0, s, Td, sp, nsep, f, xs, rc, st, host_out, dc);
    else
      launch_pdl(blk_cert_kernel<2>, dim3(cg), dim3(256), 0, s, Td, sp, nsep, f, xs, rc, st, host_out, dc);
    LAUNCH_CHECK();
    launches += 3;
  }
};

// ----------------------------------------------------------------------------
// BVP-layout BABD chain path (chain_kernels.cuh)
// ----------------------------------------------------------------------------
struct ChainSolver {
  int MB = 0;
  bool possible = false;
  const double* data = nullptr;
  const double* corner = nullptr;
  long N = 0;              // block rows after the BC row
  std::vector<long> P;     // chunks per level (P[l], l < T)
  DevBuf<double> tm, cv, glu, x1, xlev[2], xtop[2];
  bool factor_pending = false;  // lazy factor: fused into the next solve's condense pass
  std::vector<std::unique_ptr<DevBuf<double>>> phi, fl, cfl;
  DevBuf<int> cnt;
  DevBuf<unsigned> cctr;          // arrival counter of the status publish (self-resetting)
  DevStatus* host_out = nullptr;  // this solve's pinned host status slot
  int coff[kChainMaxLev + 1] = {};
  DevBuf<double> falign;
  int launches = 0;

  void init(const psg_desc& A, const Plan& Pl) {
    possible = false;
    if (A.kind != PSG_BABD || A.s != A.m || A.r != 0 || !Pl.has_corner) return;
    if (A.corner_rows != A.m || A.corner_cols != A.m) return;
    if (A.m != 2 && A.m != 4 && A.m != 8) return;
    if (reinterpret_cast<uintptr_t>(A.data) & 15) return;  // blocks arrive by 16-byte bulk copies
    MB = A.m;
    data = A.data;
    corner = A.corner;
    N = (long)A.n / MB - 1;
    if (N < 1) return;
    // chunks of kChainC0 blocks on every level (internal; independent of the
    // reference plan, whose reduced system the exact path keeps)
    P.assign(1, (N + kChainC0 - 1) / kChainC0);
    while (P.back() > kChainC0) P.push_back((P.back() + kChainC0 - 1) / kChainC0);
    const int T = (int)P.size();
    if (T > kChainMaxLev) return;
    const size_t MM = (size_t)MB * MB;
    tm.alloc((size_t)N * MM);
    cv.alloc((size_t)(N + 1) * MB);
    phi.clear();
    fl.clear();
    cfl.clear();
    fl.emplace_back(nullptr);
    cfl.emplace_back(nullptr);
    for (int l = 0; l < T; ++l) {
      phi.emplace_back(new DevBuf<double>());
      phi.back()->alloc((size_t)P[l] * MM);
      fl.emplace_back(new DevBuf<double>());
      fl.back()->alloc((size_t)(P[l] + 1) * MB);  // level l + 1
      cfl.emplace_back(new DevBuf<double>());
      cfl.back()->alloc((size_t)(P[l] + 1) * MB);
    }
    glu.alloc(MM + MB);
    x1.alloc((size_t)(P[0] + 1) * MB);
    for (int k = 0; k < 2; ++k) {
      xlev[k].alloc((size_t)(P[std::min(2, T) - 1] + 1) * MB);
      xtop[k].alloc((size_t)(P[T - 1] + 1) * MB);
    }
    int tot = 0;
    for (int l = 1; l < T; ++l) coff[l] = tot, tot += (int)P[l];
    coff[T] = tot++;
    cnt.alloc(tot);
    CUDA_TRY(cudaMemset(cnt.p, 0, sizeof(int) * tot));
    cctr.alloc(1);
    CUDA_TRY(cudaMemset(cctr.p, 0, sizeof(unsigned)));
    possible = true;
  }

  void set_data(const double* d, const double* c) {
    data = d;
    corner = c;
  }

  ChainLevelArgs args(const double* f, double* x, DevStatus* st) const {
    ChainLevelArgs g{};
    g.data = data;
    g.corner = corner;
    g.nb = (int)(N + 1);
    g.f = f;
    g.x = x;
    g.tm = tm.p;
    g.cv = cv.p;
    g.status = st;
    g.host_out = st ? host_out : nullptr;
    g.done_ctr = cctr.p;
    return g;
  }

  ChainTree tree() const {
    ChainTree t{};
    t.T = (int)P.size();
    for (int l = 0; l < t.T; ++l) {
      t.P[l] = (int)P[l];
      t.phi[l] = phi[l]->p;
      t.fl[l + 1] = fl[l + 1]->p;
      t.cfl[l + 1] = cfl[l + 1]->p;
    }
    t.cnt = cnt.p;
    for (int l = 0; l <= t.T; ++l) t.coff[l] = coff[l];
    t.glu = glu.p;
    t.x1 = x1.p;
    for (int k = 0; k < 2; ++k) {
      t.xlev[k] = xlev[k].p;
      t.xtop[k] = xtop[k].p;
    }
    return t;
  }

  template <int M, bool STORE_T, bool WITH_F>
  void fc_launch(const double* f, cudaStream_t s) {
    // m = 8: two rows per lane (half the shared-memory traffic per block;
    // bit-identical results).  PSG_CHAIN_FC1 = 1 keeps the row-per-lane kernel.
    static const bool fc1 = [] {
      const char* e = getenv("PSG_CHAIN_FC1");
      return e && atoi(e) > 0;
    }();
    if constexpr (M == 8) {
      if (!fc1) {
        constexpr int bytes2 = Fc2Cfg<M>::SMEM;
        ensure_smem(reinterpret_cast<const void*>(chain_fc2_kernel<M, STORE_T, WITH_F>), bytes2);
        const int ctas2 = (int)((P[0] + Fc2Cfg<M>::CPC - 1) / Fc2Cfg<M>::CPC);
        chain_fc2_kernel<M, STORE_T, WITH_F><<<ctas2, Fc2Cfg<M>::NW * 32, bytes2, s>>>(args(f, nullptr, nullptr), tree());
        LAUNCH_CHECK();
        ++launches;
        return;
      }
    }
    constexpr int bytes = FcCfg<M>::SMEM;
    ensure_smem(reinterpret_cast<const void*>(chain_fc_kernel<M, STORE_T, WITH_F>), bytes);
    const int ctas = (int)((P[0] + FcCfg<M>::CPC - 1) / FcCfg<M>::CPC);
    chain_fc_kernel<M, STORE_T, WITH_F><<<ctas, 128, bytes, s>>>(args(f, nullptr, nullptr), tree());
    LAUNCH_CHECK();
    ++launches;
  }

  template <int M, int KM>
  void solve_launch(const ChainLevelArgs& a, const ChainTree& t, cudaStream_t s) {
    constexpr int bytes = ChainReg<M>::SIZE * 8;
    ensure_smem(reinterpret_cast<const void*>(chain_solve_kernel<M, KM>), bytes);
    launch_pdl(chain_solve_kernel<M, KM>, dim3((unsigned)((P[0] + kChainC0 - 1) / kChainC0)), dim3(16 * M), bytes, s,
               a, t);
    LAUNCH_CHECK();
    ++launches;
  }

  template <int M>
  void down_launch(const ChainLevelArgs& a, const ChainTree& t, int sel, cudaStream_t s) {
    const int bytes = t.T * ChainReg<M>::SIZE * 8;
    ensure_smem(reinterpret_cast<const void*>(chain_down_kernel<M>), kChainMaxLev * ChainReg<M>::SIZE * 8);
    launch_pdl(chain_down_kernel<M>, dim3(t.T >= 3 ? t.P[2] : 1), dim3(32), bytes, s, a, t, sel);
    LAUNCH_CHECK();
    ++launches;
  }

  template <int M>
  void solve_t(const double* f, double* x, DevStatus* st, cudaStream_t s, cudaEvent_t* ev) {
    const ChainTree t = tree();
    if (factor_pending)  // refactor + solve: one pass over A for both
      fc_launch<M, true, true>(f, s);
    else                 // condense only (the factor of an earlier solve stays)
      fc_launch<M, false, true>(f, s);
    factor_pending = false;
    down_launch<M>(args(f, x, nullptr), t, 0, s);   // top solve, x down to level 2
    if (ev) {
      CUDA_TRY(cudaEventRecord(ev[1], s));
      CUDA_TRY(cudaEventRecord(ev[2], s));
    }
    solve_launch<M, 1>(args(f, x, nullptr), t, s);  // x through every block, separator residuals up
    down_launch<M>(args(f, x, st), t, 1, s);        // the correction down (resets the status slot)
    solve_launch<M, 2>(args(f, x, st), t, s);       // x += d, certificate
  }

  // lazy: the factor runs fused with the next solve's condense pass; force()
  // runs it alone (a caller that wants the factor data without a solve)
  void factor(cudaStream_t) { factor_pending = true; }
  void force(cudaStream_t s) {
    if (!factor_pending) return;
    if (MB == 8) fc_launch<8, true, false>(nullptr, s);
    else if (MB == 4) fc_launch<4, true, false>(nullptr, s);
    else fc_launch<2, true, false>(nullptr, s);
    factor_pending = false;
  }
  // the correction sweep resets the status slot, the correction pass publishes
  // it to the pinned host slot hout (NULL: the caller copies it)
  void solve(const double* f, double* x, DevStatus* st, cudaStream_t s, cudaEvent_t* ev, DevStatus* hout = nullptr) {
    host_out = hout;
    if (reinterpret_cast<uintptr_t>(f) & 15) {  // the passes read f by 16-byte loads
      falign.alloc((size_t)(N + 1) * MB);
      CUDA_TRY(cudaMemcpyAsync(falign.p, f, sizeof(double) * (N + 1) * MB, cudaMemcpyDeviceToDevice, s));
      f = falign.p;
    }
    if (MB == 8) solve_t<8>(f, x, st, s, ev);
    else if (MB == 4) solve_t<4>(f, x, st, s, ev);
    else solve_t<2>(f, x, st, s, ev);
  }
};

struct GenLevel {
  SMView A{};
  int es = 0, er = 0, k = 0, p = 0, q = 0;
  bool corner = false, direct = false;
  const double* f = nullptr;
  double* x = nullptr;
  std::vector<GPart> hpart;
  std::vector<int> hsep;
  DevBuf<GPart> part;
  DevBuf<int> sep;
  DevBuf<double> blocks, kr, scratch;
  DevBuf<double> Tdata, Tcorner, rhs_next, x_next;  // next level system
  DevBuf<double> work;                              // direct solve scratch
  int K = 0;                                        // direct: bordered tail size
};

constexpr int kGenDirectRows = 256;

struct GenSolver {
  std::vector<std::unique_ptr<GenLevel>> lv;
  int launches = 0;

  static Plan plan_of(const SMView& A, int p) {
    psg_desc d{A.kind, A.n, A.m, A.s, A.r, nullptr, 0, nullptr, A.cr, A.cc, 1};
    return make_plan(d, p);
  }

  void add_level(const SMView& A, int p_or_0) {
    auto L = std::make_unique<GenLevel>();
    L->A = A;
    envelope_of(A.kind, A.m, A.s, A.r, L->es, L->er);
    if (L->es + 1 + L->er > kGenMaxW) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "band envelope too wide for the GPU path"};
    if (p_or_0 == 0) {
      L->direct = true;
      L->K = 0;
      if (A.kind == PSG_BABD) L->K = std::min(A.cc + L->es + L->er, A.n);
      const long nb = A.n - L->K;
      L->work.alloc((size_t)nb * (L->es + 1 + L->er) + (size_t)nb * L->K + (size_t)A.n + (size_t)L->K * L->K +
                    (size_t)L->K + (size_t)A.n + 16);
      lv.push_back(std::move(L));
      return;
    }
    Plan P = plan_of(A, p_or_0);
    L->p = p_or_0;
    L->k = P.sep_size;
    if (L->k > kGenMaxK) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "separator block too large for the GPU path"};
    L->corner = P.has_corner;
    L->q = P.sep_count();
    L->hpart.resize(P.p);
    for (int i = 0; i < P.p; ++i) {
      const int lsi = P.has_corner ? i : i - 1, rsi = P.has_corner ? i + 1 : i;
      L->hpart[i] = GPart{P.body_begin(i), P.body_end(i) - P.body_begin(i), lsi >= 0 ? P.sep_start(lsi) : -1,
                          rsi < P.sep_count() ? P.sep_start(rsi) : -1};
    }
    L->hsep.resize(L->q);
    for (int j = 0; j < L->q; ++j) L->hsep[j] = P.sep_start(j);
    L->part.alloc(P.p);
    L->sep.alloc(L->q);
    CUDA_TRY(cudaMemcpy(L->part.p, L->hpart.data(), sizeof(GPart) * P.p, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(L->sep.p, L->hsep.data(), sizeof(int) * L->q, cudaMemcpyHostToDevice));
    const int kk = L->k * L->k;
    L->blocks.alloc((size_t)P.p * 4 * kk);
    L->kr.alloc((size_t)P.p * 2 * L->k);
    L->scratch.alloc((size_t)A.n * (L->er + 2));
    // next level: the reduced matrix as a structured matrix of q blocks of size k
    const int q = L->q, k = L->k;
    SMView T{};
    T.m = k;
    T.n = q * k;
    if (!L->corner) {
      T.kind = PSG_BLOCKTRI;
      T.s = T.r = 1;
      L->Tdata.alloc((size_t)(3 * q - 2) * kk);
    } else {
      T.kind = PSG_BABD;
      T.s = T.r = k;
      T.cr = T.cc = k;
      L->Tdata.alloc((size_t)(q >= 2 ? 2 * 2 * kk + (size_t)(q - 2) * 3 * kk : kk));
      L->Tcorner.alloc(kk);
      T.corner = L->Tcorner.p;
    }
    T.data = L->Tdata.p;
    L->rhs_next.alloc((size_t)q * k);
    L->x_next.alloc((size_t)q * k);
    lv.push_back(std::move(L));
    GenLevel& cur = *lv.back();
    // choose the next level's partition count: bodies of ~31 blocks, direct when small
    const int pn = (long)T.n > kGenDirectRows ? std::max(2, q / 32) : 0;
    (void)cur;
    add_level(T, pn);
  }

  void build(const SMView& A0, int p) {
    lv.clear();
    add_level(A0, p);
    // wire rhs/x of every level > 0
    for (size_t l = 1; l < lv.size(); ++l) {
      lv[l]->f = lv[l - 1]->rhs_next.p;
      lv[l]->x = lv[l - 1]->x_next.p;
    }
  }

  GenArgs args_of(GenLevel& L, DevStatus* st) {
    GenArgs g{};
    g.A = L.A;
    g.part = L.part.p;
    g.p = L.p;
    g.k = L.k;
    g.es = L.es;
    g.er = L.er;
    g.f = L.f;
    g.has_corner = L.corner ? 1 : 0;
    g.blocks = L.blocks.p;
    g.kr = L.kr.p;
    g.x = L.x;
    g.scratch = L.scratch.p;
    g.status = st;
    return g;
  }

  void factor(cudaStream_t s) {
    for (size_t l = 0; l + 1 < lv.size(); ++l) {
      GenLevel& L = *lv[l];
      GenArgs g = args_of(L, nullptr);
      gen_ends_kernel<0><<<2 * L.p, 32, 0, s>>>(g);
      LAUNCH_CHECK();
      const long ent = (long)L.q * L.k * L.k;
      gen_assemble_T_kernel<<<(int)((ent + 255) / 256), 256, 0, s>>>(g, L.Tdata.p, L.Tcorner.p);
      LAUNCH_CHECK();
      launches += 2;
    }
  }

  // phase 1 of level 0 alone (the reduced right-hand side into lv[0]->rhs_next)
  const double* condense(const double* f0, cudaStream_t s) {
    GenLevel& L = *lv[0];
    L.f = f0;
    GenArgs g = args_of(L, nullptr);
    gen_ends_kernel<1><<<2 * L.p, 32, 0, s>>>(g);
    LAUNCH_CHECK();
    const long ent = (long)L.q * L.k;
    gen_assemble_rhs_kernel<<<(int)((ent + 255) / 256), 256, 0, s>>>(g, L.sep.p, L.rhs_next.p);
    LAUNCH_CHECK();
    return L.rhs_next.p;
  }

  void solve(const double* f0, double* x0, DevStatus* st, cudaStream_t s, cudaEvent_t* ev, size_t from = 0) {
    lv[from]->f = f0;
    lv[from]->x = x0;
    for (size_t l = from; l + 1 < lv.size(); ++l) {
      GenLevel& L = *lv[l];
      GenArgs g = args_of(L, l == 0 ? st : nullptr);
      gen_ends_kernel<1><<<2 * L.p, 32, 0, s>>>(g);
      LAUNCH_CHECK();
      const long ent = (long)L.q * L.k;
      gen_assemble_rhs_kernel<<<(int)((ent + 255) / 256), 256, 0, s>>>(g, L.sep.p, L.rhs_next.p);
      LAUNCH_CHECK();
      launches += 2;
      if (l == from && ev) CUDA_TRY(cudaEventRecord(ev[1], s));
    }
    for (size_t l = lv.size(); l-- > from;) {
      GenLevel& L = *lv[l];
      if (l == from && ev) CUDA_TRY(cudaEventRecord(ev[2], s));
      if (L.direct) {
        gen_direct_kernel<<<1, 32, 0, s>>>(L.A, L.es, L.er, L.K, L.f, L.x, L.work.p, l == 0 ? st : nullptr);
        LAUNCH_CHECK();
        launches += 1;
        continue;
      }
      GenArgs g = args_of(L, l == 0 ? st : nullptr);
      g.xsep = L.x_next.p;
      if (!blk_backsolve(L, g, s)) {
        gen_backsolve_kernel<<<L.p, 32, 0, s>>>(g);
        LAUNCH_CHECK();
      }
      launches += 1;
    }
  }

  // K x K block-tridiagonal levels (BlockTridiagonal m = K, Banded s, r <= K
  // with separators of K rows) whose bodies fit one warp go through the block
  // body kernel (blk_kernels.cuh) instead of the band back-substitution.
  bool blk_backsolve(const GenLevel& L, const GenArgs& g, cudaStream_t s) {
    static const bool off = getenv("PSG_NO_BLK") != nullptr;
    if (off || L.corner || L.k < 2 || L.k > 4) return false;
    int layout;
    if (L.A.kind == PSG_BLOCKTRI && L.A.m == L.k)
      layout = kBlkBlockTri;
    else if (L.A.kind == PSG_BANDED && L.A.s <= L.k && L.A.r <= L.k)
      layout = kBlkBanded;
    else
      return false;
    int maxL = 0, minL = INT_MAX;
    for (const GPart& P : L.hpart) {
      maxL = std::max(maxL, P.L);
      minL = std::min(minL, P.L);
    }
    if (minL < 2 * L.k) return false;
    BlkArgs a{};
    a.data = L.A.data;
    a.n = L.A.n;
    a.s = L.A.s;
    a.r = L.A.r;
    a.f = g.f;
    a.x = g.x;
    a.xsep = g.xsep;
    a.part = g.part;
    a.nseg = L.p;
    a.rec = nullptr;
    a.status = g.status;
    fill_band_offsets(a, L.k, L.A.n, L.A.s, L.A.r,
                      layout == kBlkBanded ? (size_t)body_entry_count(PSG_BANDED, L.A.n, 1, L.A.s, L.A.r)
                                           : (size_t)(3 * (L.A.n / L.k) - 2) * L.k * L.k);
    return launch_blk_segments(L.k, (maxL + L.k - 1) / L.k, layout, a, s);
  }

  void restore_level1_wiring() {
    if (lv.size() > 1) {
      lv[1]->f = lv[0]->rhs_next.p;
      lv[1]->x = lv[0]->x_next.p;
    }
  }
};

}  // namespace

// ----------------------------------------------------------------------------
// the handle
// ----------------------------------------------------------------------------
// ----------------------------------------------------------------------------
// Pivoting strategies (LuPivot / Qr) and the circulant-like kind
// (piv_kernels.cuh): one warp per body, adaptive extras, the reduced band
// factored by the same engine in dense-LU mode.
// ----------------------------------------------------------------------------
struct PivRecBuf {
  DevBuf<int4> meta;
  DevBuf<unsigned char> tslot, aslot;
  DevBuf<double> mu, av, tau, urow, uspk;
  PivRec view{};
  void alloc(size_t steps, int NT, int NA, int URW, int NS) {
    meta.alloc(steps);
    tslot.alloc(steps * NT);
    mu.alloc(steps * NT);
    aslot.alloc(steps * NA);
    av.alloc(steps * NA);
    tau.alloc(steps);
    urow.alloc(steps * URW);
    uspk.alloc(steps * NS);
    view = PivRec{meta.p, tslot.p, mu.p, aslot.p, av.p, tau.p, urow.p, uspk.p, NT, NA, URW, NS};
  }
};

struct PivSolver {
  SMView A{};  // canonical matrix (circulant-like: rows rotated)
  Plan P;
  int p = 0, k = 0, es = 0, er = 0, strategy = kPvPartial, cap = 0, KD = 0;
  double tol = 1e-8;
  bool corner = false;
  std::vector<GPart> hpart;
  DevBuf<GPart> part;
  PivRecBuf rb, rr_rec;
  DevBuf<double> kept;
  DevBuf<int> ndef, xpos, status, koff;
  std::vector<int> hndef, hxpos, hkoff;
  // the reduced system
  int dim = 0, w = 0, kb = 0, q = 0;
  std::vector<int> rpos, rsize;  // position order: global start, size (k or 1)
  DevBuf<double> rband, rborder;
  // solve scratch
  DevBuf<double> ghat, kr, rrhs, xk, rghat;
  int launches = 0;

  static size_t smem_bytes() { return sizeof(PivSmem); }

  PivArgs args() const {
    PivArgs a{};
    a.A = A;
    a.part = part.p;
    a.p = p;
    a.k = k;
    a.es = es;
    a.er = er;
    a.strategy = strategy;
    a.tol = tol;
    a.cap = cap;
    a.KD = KD;
    a.kept = kept.p;
    a.ndef = ndef.p;
    a.xpos = xpos.p;
    a.rband = rband.p;
    a.rborder = rborder.p;
    a.dim = dim;
    a.w = w;
    a.kb = kb;
    a.rec = rb.view;
    a.status = status.p;
    a.ghat = ghat.p;
    a.kr = kr.p;
    a.xk = xk.p;
    a.koff = koff.p;
    return a;
  }

  void init(const SMView& Av, const Plan& plan, int strat, double tol_) {
    A = Av;
    P = plan;
    p = plan.p;
    k = plan.sep_size;
    corner = plan.has_corner;
    strategy = strat;
    tol = tol_;
    envelope_of(A.kind == PSG_CIRCULANT ? PSG_BANDED : A.kind, A.m, A.s, A.r, es, er);
    if (es + er + 1 > kPvRing || es > 31)
      throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "band envelope too wide for the pivoting GPU path"};
    if (k > kGenMaxK) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "separator block too large for the pivoting GPU path"};
    cap = std::min({16, kPvSpk - 2 * k, kPvSlots - 1 - es - 2 * k});
    if (strategy == kPvNoPivot) cap = std::max(cap, 1);
    if (cap < 1) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "no room for deferred pivots in the pivoting GPU path"};
    KD = 2 * k + cap;
    hpart.resize(p);
    for (int i = 0; i < p; ++i) {
      const int lsi = corner ? i : i - 1, rsi = corner ? i + 1 : i;
      hpart[i] = GPart{plan.body_begin(i), plan.body_end(i) - plan.body_begin(i), lsi >= 0 ? plan.sep_start(lsi) : -1,
                       rsi < plan.sep_count() ? plan.sep_start(rsi) : -1};
    }
    part.alloc(p);
    CUDA_TRY(cudaMemcpy(part.p, hpart.data(), sizeof(GPart) * p, cudaMemcpyHostToDevice));
    rb.alloc((size_t)A.n, es + 2 * k + cap, es + 1, es + er + 1, 2 * k + cap);
    kept.alloc((size_t)p * KD * KD);
    ndef.alloc(p);
    xpos.alloc((size_t)p * cap);
    status.alloc(4);
    koff.alloc(p);
    ghat.alloc(A.n);
    kr.alloc((size_t)p * KD);
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_done[dev & 63]) {
      CUDA_TRY(cudaFuncSetAttribute(piv_factor_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes()));
      CUDA_TRY(cudaFuncSetAttribute(piv_factor_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes()));
      attr_done[dev & 63] = true;
    }
  }

  void check_status(cudaStream_t s) {
    int st[4];
    CUDA_TRY(cudaMemcpyAsync(st, status.p, sizeof st, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (st[2] != INT_MAX)
      throw Fail{PSG_E_ZERO_PIVOT, "partition " + std::to_string(st[2] + 1) + ": zero pivot in the no-pivot elimination"};
    if (st[1] != INT_MAX)
      throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "partition " + std::to_string(st[1] + 1) + ": more than " +
                                                 std::to_string(cap) + " deferred pivots in one body"};
    if (st[0] != INT_MAX)
      throw Fail{PSG_E_EXHAUSTED_BODY, "partition " + std::to_string(st[0] + 1) +
                                          ": every pivot deferred; body is structurally degenerate"};
    if (st[3] != INT_MAX) throw Fail{PSG_E_SINGULAR_REDUCED_SYSTEM, "reduced system is singular"};
  }

  void reset_status(cudaStream_t s) {
    const int init[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
    CUDA_TRY(cudaMemcpyAsync(status.p, init, sizeof init, cudaMemcpyHostToDevice, s));
  }

  void factor(cudaStream_t s) {
    launches = 0;
    reset_status(s);
    PivArgs a = args();
    piv_factor_kernel<0><<<p, 32, smem_bytes(), s>>>(a);
    LAUNCH_CHECK();
    ++launches;
    hndef.resize(p);
    hxpos.resize((size_t)p * cap);
    CUDA_TRY(cudaMemcpyAsync(hndef.data(), ndef.p, sizeof(int) * p, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(hxpos.data(), xpos.p, sizeof(int) * hxpos.size(), cudaMemcpyDeviceToHost, s));
    check_status(s);
    // reduced layout in position order (src/parfact.cpp:72-88): separators and extras
    rpos.clear();
    rsize.clear();
    hkoff.assign(p, 0);
    int maxkd = 1;
    auto add_sep = [&](int j) {
      rpos.push_back(P.sep_start(j));
      rsize.push_back(k);
    };
    int off = 0;
    std::vector<int> sepoff(P.sep_count());
    if (corner) {
      sepoff[0] = 0;
      add_sep(0);
      off = k;
    }
    for (int i = 0; i < p; ++i) {
      const int k0 = hpart[i].ls >= 0 ? k : 0, k1 = hpart[i].rs >= 0 ? k : 0;
      hkoff[i] = off - k0;
      for (int e = 0; e < hndef[i]; ++e) {
        rpos.push_back(hpart[i].b + hxpos[(size_t)i * cap + e]);
        rsize.push_back(1);
      }
      off += hndef[i];
      if (k1) {
        const int j = corner ? i + 1 : i;
        sepoff[j] = off;
        add_sep(j);
        off += k;
      }
      maxkd = std::max(maxkd, k0 + hndef[i] + k1);
    }
    dim = off;
    q = (int)rpos.size();
    w = maxkd - 1;
    kb = corner ? k : 0;
    CUDA_TRY(cudaMemcpyAsync(koff.p, hkoff.data(), sizeof(int) * p, cudaMemcpyHostToDevice, s));
    rband.alloc((size_t)dim * (2 * w + 1));
    rborder.alloc((size_t)dim * std::max(kb, 1));
    CUDA_TRY(cudaMemsetAsync(rband.p, 0, sizeof(double) * (size_t)dim * (2 * w + 1), s));
    CUDA_TRY(cudaMemsetAsync(rborder.p, 0, sizeof(double) * (size_t)dim * std::max(kb, 1), s));
    a = args();
    piv_assemble_kernel<0><<<p, 32, 0, s>>>(a);
    LAUNCH_CHECK();
    piv_assemble_kernel<1><<<p, 32, 0, s>>>(a);
    LAUNCH_CHECK();
    launches += 2;
    // the reduced LU with partial pivoting (src/parfact.cpp:134-166)
    rr_rec.alloc((size_t)dim, w + 1, 1, 2 * w + 1, std::max(kb, 1));
    rrhs.alloc(dim);
    xk.alloc(dim);
    rghat.alloc(dim);
    a = args();
    a.rec = rr_rec.view;
    piv_factor_kernel<1><<<1, 32, smem_bytes(), s>>>(a);
    LAUNCH_CHECK();
    ++launches;
    check_status(s);
  }

  PivArgs reduced_args(const double* r, double* x) const {
    PivArgs a = args();
    a.rec = rr_rec.view;
    a.rr = r;
    a.xk = x;
    a.ghat = rghat.p;
    return a;
  }

  void solve(const double* df, double* dx, cudaStream_t s, cudaEvent_t* ev) {
    PivArgs a = args();
    a.f = df;
    a.x = dx;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
    piv_condense_kernel<<<p, 32, 0, s>>>(a);
    LAUNCH_CHECK();
    piv_rrhs_kernel<<<p, 32, 0, s>>>(a, rrhs.p);
    LAUNCH_CHECK();
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], s));
    piv_reduced_solve_kernel<<<1, 32, 0, s>>>(reduced_args(rrhs.p, xk.p));
    LAUNCH_CHECK();
    if (ev) CUDA_TRY(cudaEventRecord(ev[2], s));
    piv_backsolve_kernel<<<p, 32, 0, s>>>(a);
    LAUNCH_CHECK();
    if (ev) CUDA_TRY(cudaEventRecord(ev[3], s));
    launches = 4;
  }

  void solve_reduced(const double* r, double* x, cudaStream_t s) {
    piv_reduced_solve_kernel<<<1, 32, 0, s>>>(reduced_args(r, x));
    LAUNCH_CHECK();
  }

  // exact operation count of the reference's dense reduced LU (src/parfact.cpp:134-184)
  long long reduced_ops() const {
    const long long n = dim;
    return 3 * (n * (n - 1) / 2) + (n - 1) * n * (2 * n - 1) / 6 + n;
  }

  void dense_T(double* T) const {
    std::vector<double> band((size_t)dim * (2 * w + 1)), border((size_t)dim * std::max(kb, 1));
    CUDA_TRY(cudaMemcpy(band.data(), rband.p, sizeof(double) * band.size(), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(border.data(), rborder.p, sizeof(double) * border.size(), cudaMemcpyDeviceToHost));
    std::fill(T, T + (size_t)dim * dim, 0.0);
    for (int r = 0; r < dim; ++r) {
      for (int d = 0; d <= 2 * w; ++d) {
        const int c = r - w + d;
        if (c >= 0 && c < dim - kb) T[(size_t)r * dim + c] = band[(size_t)r * (2 * w + 1) + d];
      }
      for (int u = 0; u < kb; ++u) T[(size_t)r * dim + (dim - kb + u)] = border[(size_t)r * kb + u];
    }
  }
};

struct psg_handle {
  int device = 0;  // where the factorization lives (DeviceGuard in every entry point)
  psg_desc A{};    // device view
  Plan plan;
  int strategy = 0;
  DevBuf<double> own_data, own_corner;
  TriSolver tri;
  GenSolver gen;
  BlkSolver blk;                        // speculative path of the K x K block kinds
  ChainSolver chain;                    // BVP-layout BABD chain path
  std::unique_ptr<PivSolver> piv;       // LuPivot / Qr, and every strategy of the circulant-like kind
  int rot = 0;                          // circulant-like: rows rotated down by rot (permute_corner)
  DevBuf<double> d_fperm;               // rotated rhs
  bool generic = false;                 // non-tridiagonal kinds: generic exact path
  double refine_tol = 1e-14;            // generic path: refine once when ||Ax-f||/||f|| exceeds this
  double last_residual = 0.0;
  DevBuf<double> d_r, d_d;              // refinement residual / correction
  DevBuf<unsigned long long> d_norm;
  std::vector<int> seg_start, seg_len;  // level-0 segmentation when refined
  bool refined = false;
  const double* gen_ref_data = nullptr;  // refined tridiagonal: gen holds the reference plan's reduced system
  bool gen_ref_factored = false;
  // options
  bool speculative = true;
  double cert_tol = 1e-14;
  // state: which factor data is current
  bool spec_factored = false, exact_factored = false;
  DevBuf<DevStatus> d_status;
  DevStatus* h_status = nullptr;  // pinned slot
  DevBuf<double> d_f, d_x;        // host-path staging
  std::vector<cudaEvent_t> host_evs;  // host-path chunk events
  cudaEvent_t ev_f0 = nullptr, ev_f1 = nullptr, ev_done = nullptr, ev[4] = {};
  std::mutex mu;
  int factor_launches = 0, solve_launches = 0;
  // asynchronous solves: per-solve status slots, repaired at psg_sync
  static constexpr int kRing = 64;
  struct Pending {
    int slot;
    const double* f;
    double* x;
    cudaStream_t s;
    bool spec, timing;
    int launches;
  };
  std::vector<Pending> pending;
  psg_stats carried{};      // statistics of solves drained by psg_refactor, reported at the next psg_sync
  bool has_carried = false;
  cudaStream_t last_stream = nullptr;  // stream of the last enqueued work (see order_on)
  bool used = false;
  DevBuf<DevStatus> d_ring;
  DevStatus* h_ring = nullptr;               // pinned mirror
  cudaEvent_t ring_done[kRing] = {}, ring_t[kRing][4] = {};
  long async_count = 0;
  ~psg_handle() {
    if (ev_done) cudaEventSynchronize(ev_done);  // buffers go back to the cache only when idle
    for (auto& pd : pending) cudaEventSynchronize(ring_done[pd.slot]);
    for (cudaEvent_t e : {ev_f0, ev_f1, ev_done, ev[0], ev[1], ev[2], ev[3]})
      if (e) event_pool().put(e);
    for (int i = 0; i < kRing; ++i) {
      if (ring_done[i]) event_pool().put(ring_done[i]);
      for (int j = 0; j < 4; ++j)
        if (ring_t[i][j]) event_pool().put(ring_t[i][j]);
    }
    for (cudaEvent_t e : host_evs) event_pool().put(e);
    if (h_status) pinned_slots().put(h_status);
    if (h_ring) cudaFreeHost(h_ring);
  }
  bool use_spec() const { return !generic && speculative && tri.spec_possible(); }
  bool use_blk() const { return generic && speculative && blk.possible; }
  bool use_chain() const { return generic && speculative && chain.possible; }
  bool spec_mode() const { return generic ? (use_blk() || use_chain()) : use_spec(); }
};

namespace {

// The reference layout data = [sub (n-1) | diag (n) | super (n-1)]
// (src/structmat.cpp:33-38): a_r = data[r-1], b_r = data[n-1+r],
// c_r = data[2n-1+r]; any row index whose address stays inside data is safe
// to over-read (the staging widens copies to 16-byte boundaries).
TriRows tri_rows(const psg_desc& A) {
  const double* d = A.data;
  const long n = A.n;
  return TriRows{make_rows(d - 1, 1, (int)n, 1, 3 * n - 1), make_rows(d + (n - 1), 0, (int)n, -(n - 1), 2 * n - 1),
                 make_rows(d + (2 * n - 1), 0, (int)n - 1, -(2 * n - 1), n - 1)};
}

// Level-0 segmentation: the reference bodies, refined (extra one-row
// separators inside a body) when a body exceeds one warp's capacity.
SegMap plan_segments(const Plan& P, std::vector<int>& st, std::vector<int>& ln, bool& refined, int& maxlen,
                     int& minlen) {
  st.clear();
  ln.clear();
  refined = false;
  maxlen = int(P.base + (P.rem ? 1 : 0));
  minlen = int(P.base);
  // few long bodies (small p): optionally split them further so that K3
  // gets more warps (PSG_SEG_TARGET = segments wanted; off by default:
  // config 0 measured 0.056-0.060 ms/step with targets 1, 2048 and 4096)
  static const int target = [] {
    const char* e = getenv("PSG_SEG_TARGET");
    return e ? atoi(e) : 0;
  }();
  int par = 1;
  if (P.p < target && (long)P.p * maxlen >= (1L << 18))
    par = std::max(1, std::min((target + P.p - 1) / P.p, minlen / 256));
  if (maxlen <= kMaxSeg && par == 1) return SegMap{P.p, int(P.base), int(P.rem), nullptr, nullptr};
  refined = true;
  maxlen = 0;
  minlen = INT_MAX;
  for (int i = 0; i < P.p; ++i) {
    const int b = P.body_begin(i), L = P.body_end(i) - b;
    const int t = std::max(par, (L + 1 + kMaxSeg) / (kMaxSeg + 1));  // sub-bodies
    const long body = (long)L - (t - 1);
    const long base = body / t, rem = body % t;
    long cur = b;
    for (int u = 0; u < t; ++u) {
      const long len = base + (u < rem ? 1 : 0);
      st.push_back(int(cur));
      ln.push_back(int(len));
      maxlen = std::max<int>(maxlen, int(len));
      minlen = std::min<int>(minlen, int(len));
      cur += len + 1;
    }
  }
  return SegMap{(int)st.size(), 0, 0, nullptr, nullptr};
}

void check_strategy(const psg_desc& A, int strategy) {
  switch (strategy) {
    case PSG_LU:
    case PSG_LUD: return;
    case PSG_CR:
      // strategy_supports (src/localfact.cpp:31-42)
      if (A.kind == PSG_BLOCKTRI || (A.kind == PSG_BANDED && A.s == 1 && A.r == 1)) return;
      throw Fail{PSG_E_UNSUPPORTED_KIND, "strategy cr does not support this kind"};
    case PSG_ARCE:
      if (A.kind != PSG_ABD && A.kind != PSG_BABD)
        throw Fail{PSG_E_UNSUPPORTED_KIND, "strategy arce does not support this kind"};
      throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "strategy arce has no GPU path"};
    case PSG_LUPIVOT:
    case PSG_QR: return;  // every kind (src/localfact.cpp:31-42)
    default: throw Fail{PSG_E_INVALID_PARAMETER, "unknown strategy"};
  }
}

bool is_tridiag(const psg_desc& A) { return A.kind == PSG_BANDED && A.s == 1 && A.r == 1; }

// (Re)compute the factor data for the current mode.
// Calls on one handle may come from different streams; they share the
// handle's scratch (status words, staging, reduced-system buffers), so a
// stream that differs from the previous call's first waits for the work
// already enqueued on the handle (ev_done is recorded at the end of every
// entry point).
void order_on(psg_handle* h, cudaStream_t s) {
  if (h->used && s != h->last_stream) CUDA_TRY(cudaStreamWaitEvent(s, h->ev_done, 0));
  h->last_stream = s;
  h->used = true;
}

void run_factor(psg_handle* h, cudaStream_t s) {
  h->tri.launches = 0;
  CUDA_TRY(cudaEventRecord(h->ev_f0, s));
  if (h->piv) {
    h->piv->factor(s);
    h->spec_factored = h->exact_factored = true;
    h->factor_launches = h->piv->launches;
    CUDA_TRY(cudaEventRecord(h->ev_f1, s));
    return;
  }
  if (h->generic) {
    h->gen.launches = 0;
    h->blk.launches = 0;
    if (h->use_blk()) {
      h->blk.spec_factor(s);
      h->spec_factored = true;
      h->factor_launches = h->blk.launches;
    } else if (h->use_chain()) {
      h->chain.launches = 0;
      h->chain.factor(s);
      h->spec_factored = true;
      h->factor_launches = h->chain.launches;
    } else {
      h->gen.factor(s);
      h->exact_factored = true;
      h->factor_launches = h->gen.launches;
    }
    CUDA_TRY(cudaEventRecord(h->ev_f1, s));
    return;
  }
  if (h->use_spec()) {
    h->tri.spec_factor(s);
    h->spec_factored = true;
  } else {
    h->tri.exact_factor(s);
    h->exact_factored = true;
  }
  CUDA_TRY(cudaEventRecord(h->ev_f1, s));
  h->factor_launches = h->tri.launches;
}

int partition_of_segment(const psg_handle* h, int seg) {
  if (!h->refined) return seg + 1;
  const int row = h->seg_start[std::min<size_t>(seg, h->seg_start.size() - 1)];
  int lo = 0, hi = h->plan.p - 1;  // last partition whose body begins at or before row
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (h->plan.body_begin(mid) <= row)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo + 1;
}

}  // namespace

extern "C" {

#ifndef PSG_SOURCE_HASH
#define PSG_SOURCE_HASH "unknown"
#endif
const char* psg_version(void) { return "psg-b200 0.3 (sm_100a) src " PSG_SOURCE_HASH; }

int psg_config_shape(int cfg, int size, int* kind, int* n, int* m, int* s, int* r, size_t* data_len,
                     int* corner_rows, int* corner_cols) {
  int K, N, Mm, S, R, cr = 0, cc = 0;
  switch (cfg) {
    case 0:
    case 1: K = PSG_BANDED; N = size; Mm = 1; S = 1; R = 1; break;
    case 2: K = PSG_BLOCKTRI; N = 4 * size; Mm = 4; S = 1; R = 1; break;
    case 3: K = PSG_BANDED; N = size; Mm = 1; S = 3; R = 3; break;
    case 4: K = PSG_BABD; N = 8 * (size + 1); Mm = 8; S = 8; R = 0; cr = cc = 8; break;
    default: return 1 + PSG_E_INVALID_PARAMETER;
  }
  if (kind) *kind = K;
  if (n) *n = N;
  if (m) *m = Mm;
  if (s) *s = S;
  if (r) *r = R;
  if (corner_rows) *corner_rows = cr;
  if (corner_cols) *corner_cols = cc;
  if (data_len) *data_len = body_entry_count(K, N, Mm, S, R);
  return 0;
}

int psg_generate_config(int cfg, int size, uint64_t seed, double* data, double* corner, double* f, void* stream,
                        char* err, size_t errlen) {
  try {
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = 148 * 8, tpb = 256;
    switch (cfg) {
      case 0:
      case 1: gen_tridiag_kernel<<<grid, tpb, 0, s>>>(seed, size, data, f); break;
      case 2: gen_blocktri_kernel<<<grid, tpb, 0, s>>>(seed, size, data, f); break;
      case 3: gen_banded7_kernel<<<grid, tpb, 0, s>>>(seed, size, data, f); break;
      case 4: gen_babd_kernel<<<grid, tpb, 0, s>>>(seed, size, data, corner, f); break;
      default: throw Fail{PSG_E_INVALID_PARAMETER, "unknown config"};
    }
    LAUNCH_CHECK();
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_plan(const psg_desc* A, int p, int* body_begin, int* body_end, int* sep_start, int* sep_count,
             int* sep_size, char* err, size_t errlen) {
  try {
    validate(*A);
    Plan P = make_plan(*A, p);
    for (int i = 0; i < p; ++i) {
      body_begin[i] = P.body_begin(i);
      body_end[i] = P.body_end(i);
    }
    for (int j = 0; j < P.sep_count(); ++j) sep_start[j] = P.sep_start(j);
    *sep_count = P.sep_count();
    *sep_size = P.sep_size;
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

// Device copy of A for a pivoting handle; circulant-like rows rotated down by
// r so all wrap content sits in the upper-right corner (permute_corner,
// src/partition.cpp:175-202): the canonical matrix has bandwidths (s + r, 0).
void piv_set_matrix(psg_handle* h, const psg_desc& Ain, cudaStream_t s) {
  h->A = Ain;
  const double* src = Ain.data;
  DevBuf<double> staged;
  if (!Ain.on_device) {
    (Ain.kind == PSG_CIRCULANT && Ain.r > 0 ? staged : h->own_data).alloc(Ain.data_len);
    double* dst = Ain.kind == PSG_CIRCULANT && Ain.r > 0 ? staged.p : h->own_data.p;
    CUDA_TRY(cudaMemcpyAsync(dst, Ain.data, sizeof(double) * Ain.data_len, cudaMemcpyHostToDevice, s));
    src = dst;
    h->A.data = dst;
    if (Ain.corner) {
      const size_t cn = (size_t)Ain.corner_rows * Ain.corner_cols;
      h->own_corner.alloc(cn);
      CUDA_TRY(cudaMemcpyAsync(h->own_corner.p, Ain.corner, sizeof(double) * cn, cudaMemcpyHostToDevice, s));
      h->A.corner = h->own_corner.p;
    }
    h->A.on_device = 1;
  }
  h->rot = 0;
  if (Ain.kind == PSG_CIRCULANT && Ain.r > 0) {
    h->own_data.alloc(Ain.data_len);
    piv_rotate_kernel<<<148 * 8, 256, 0, s>>>(Ain.n, Ain.s + Ain.r + 1, Ain.r, src, h->own_data.p);
    LAUNCH_CHECK();
    h->A.data = h->own_data.p;
    h->A.s = Ain.s + Ain.r;
    h->A.r = 0;
    h->rot = Ain.r;
    CUDA_TRY(cudaStreamSynchronize(s));  // staged source goes back to the cache
  }
}

int piv_strategy_of(int strategy) {
  return strategy == PSG_LUPIVOT ? kPvPartial : strategy == PSG_QR ? kPvQr : kPvNoPivot;
}

int psg_factor(const psg_desc* Ain, int p, int strategy, double tol, void* stream, psg_handle** out, char* err,
               size_t errlen) {
  *out = nullptr;
  try {
    std::unique_ptr<psg_handle> h(new psg_handle);
    CUDA_TRY(cudaGetDevice(&h->device));
    validate(*Ain);
    check_strategy(*Ain, strategy);
    if (strategy == PSG_LUPIVOT || strategy == PSG_QR || Ain->kind == PSG_CIRCULANT) {
      cudaStream_t s = (cudaStream_t)stream;
      for (cudaEvent_t* e : {&h->ev_f0, &h->ev_f1, &h->ev_done, &h->ev[0], &h->ev[1], &h->ev[2], &h->ev[3]})
        *e = event_pool().get();
      h->strategy = strategy;
      piv_set_matrix(h.get(), *Ain, s);
      h->plan = make_plan(h->A, p);
      h->generic = true;
      CUDA_TRY(cudaStreamSynchronize(s));
      h->piv = std::make_unique<PivSolver>();
      SMView V{h->A.kind, h->A.n, h->A.m, h->A.s, h->A.r, h->A.data, h->A.corner, h->A.corner_rows, h->A.corner_cols};
      h->piv->init(V, h->plan, piv_strategy_of(strategy), tol);
      h->d_status.alloc(1);
      h->h_status = static_cast<DevStatus*>(pinned_slots().get());
      run_factor(h.get(), s);
      CUDA_TRY(cudaEventRecord(h->ev_done, s));
      h->last_stream = s;
      h->used = true;
      *out = h.release();
      return 0;
    }
    h->plan = make_plan(*Ain, p);
    h->generic = !is_tridiag(*Ain);
    cudaStream_t s = (cudaStream_t)stream;
    for (cudaEvent_t* e : {&h->ev_f0, &h->ev_f1, &h->ev_done, &h->ev[0], &h->ev[1], &h->ev[2], &h->ev[3]})
      *e = event_pool().get();
    h->A = *Ain;
    h->strategy = strategy;
    if (!Ain->on_device) {
      h->own_data.alloc(Ain->data_len);
      CUDA_TRY(cudaMemcpyAsync(h->own_data.p, Ain->data, sizeof(double) * Ain->data_len, cudaMemcpyHostToDevice, s));
      h->A.data = h->own_data.p;
      if (Ain->corner) {
        const size_t cn = (size_t)Ain->corner_rows * Ain->corner_cols;
        h->own_corner.alloc(cn);
        CUDA_TRY(cudaMemcpyAsync(h->own_corner.p, Ain->corner, sizeof(double) * cn, cudaMemcpyHostToDevice, s));
        h->A.corner = h->own_corner.p;
      }
      h->A.on_device = 1;
    }
    if (h->generic) {
      SMView V{h->A.kind, h->A.n, h->A.m, h->A.s, h->A.r, h->A.data, h->A.corner, h->A.corner_rows, h->A.corner_cols};
      CUDA_TRY(cudaStreamSynchronize(s));  // plan uploads below use the legacy stream
      h->gen.build(V, p);
      h->blk.init(h->A, h->plan);
      h->chain.init(h->A, h->plan);
    } else {
      int maxlen = 0, minlen = 0;
      SegMap S0 = plan_segments(h->plan, h->seg_start, h->seg_len, h->refined, maxlen, minlen);
      h->tri.init(tri_rows(h->A), h->A.n, S0, maxlen, minlen, h->refined ? &h->seg_start : nullptr,
                  h->refined ? &h->seg_len : nullptr, s);
    }
    h->d_status.alloc(1);
    h->h_status = static_cast<DevStatus*>(pinned_slots().get());
    run_factor(h.get(), s);
    CUDA_TRY(cudaEventRecord(h->ev_done, s));
    h->last_stream = s;
    h->used = true;
    *out = h.release();
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

void psg_release(psg_handle* h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  delete h;
}

int psg_set_option(psg_handle* h, int option, double value) {
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    switch (option) {
      case PSG_OPT_SPECULATIVE:
        h->speculative = value != 0.0;
        if ((h->spec_mode() && !h->spec_factored) || (!h->spec_mode() && !h->exact_factored)) {
          run_factor(h, h->last_stream);
          CUDA_TRY(cudaEventRecord(h->ev_done, h->last_stream));
        }
        break;
      case PSG_OPT_HALO:
        if ((int)value != kHalo) return 1 + PSG_E_INVALID_PARAMETER;  // fixed to the warp width
        break;
      case PSG_OPT_CERT_TOL: h->cert_tol = value; break;
      case PSG_OPT_BODY_CERT: h->tri.body_cert = value != 0.0; break;
      default: return 1 + PSG_E_INVALID_PARAMETER;
    }
  } catch (const Fail& f_) {
    return 1 + f_.code;
  }
  return 0;
}

int psg_factor_wait(const psg_handle* hc, double* device_seconds) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  if (cudaEventSynchronize(h->ev_f1) != cudaSuccess) return 1 + PSG_E_CUDA;
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, h->ev_f0, h->ev_f1) != cudaSuccess) ms = 0.f;
  if (device_seconds) *device_seconds = 1e-3 * ms;
  return 0;
}

int psg_last_launches(const psg_handle* h, int* f, int* s) {
  if (f) *f = h->factor_launches;
  if (s) *s = h->solve_launches;
  return 0;
}

namespace {

// Generic (non-tridiagonal) solve: exact, certified by its residual, refined
// once when the residual exceeds refine_tol.  Blocking.
int generic_solve(psg_handle* h, const double* df, double* dx, cudaStream_t s, bool timing, double* cert) {
  const int n = h->A.n;
  for (int i = 0; i < kCertSlots; ++i) h->h_status->cert_bits[i] = 0ull;
  h->h_status->bad_seg = INT_MAX;
  h->h_status->pivot_seg = INT_MAX;
  CUDA_TRY(cudaMemcpyAsync(h->d_status.p, h->h_status, sizeof(DevStatus), cudaMemcpyHostToDevice, s));
  if (timing) CUDA_TRY(cudaEventRecord(h->ev[0], s));
  h->gen.launches = 0;
  h->gen.solve(df, dx, h->d_status.p, s, timing ? h->ev : nullptr);
  if (timing) CUDA_TRY(cudaEventRecord(h->ev[3], s));
  MatView v{h->A.kind, h->A.n, h->A.m, h->A.s, h->A.r, h->A.data, h->A.corner, h->A.corner_rows, h->A.corner_cols};
  h->d_r.alloc(n);
  h->d_norm.alloc(2);
  auto resid = [&]() {
    unsigned long long hb[2];
    CUDA_TRY(cudaMemsetAsync(h->d_norm.p, 0, 2 * sizeof(unsigned long long), s));
    residual_vec_kernel<<<148 * 8, 256, 0, s>>>(v, dx, df, h->d_r.p, h->d_norm.p);
    LAUNCH_CHECK();
    CUDA_TRY(cudaMemcpyAsync(hb, h->d_norm.p, sizeof hb, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(h->h_status, h->d_status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const double num = bits_to_double(hb[0]), den = bits_to_double(hb[1]);
    return den > 0 ? num / den : num;
  };
  double rel = resid();
  int launches = h->gen.launches + 1;
  const DevStatus st0 = *h->h_status;
  if (st0.pivot_seg != INT_MAX)
    throw Fail{PSG_E_ZERO_PIVOT, "partition " + std::to_string(st0.pivot_seg + 1) + ": zero pivot in the no-pivot elimination"};
  if (rel > h->refine_tol && rel == rel) {
    h->d_d.alloc(n);
    h->gen.launches = 0;
    h->gen.solve(h->d_r.p, h->d_d.p, nullptr, s, nullptr);
    axpy_kernel<<<148 * 8, 256, 0, s>>>(n, h->d_d.p, dx);
    LAUNCH_CHECK();
    launches += h->gen.launches + 2;
    rel = resid();
  }
  h->gen.lv[0]->f = df;
  h->gen.lv[0]->x = dx;
  if (!(rel == rel) || st0.bad_seg != INT_MAX)
    throw Fail{PSG_E_SINGULAR_REDUCED_SYSTEM, "non-finite solution: the reduced system is singular"};
  *cert = rel;
  return launches;
}

struct Outcome {
  double cert = 0;
  bool bad = false, pivot = false;
  int pivot_seg = 0;
};

Outcome read_status(const DevStatus& st) {
  Outcome o;
  for (int i = 0; i < kCertSlots; ++i) o.cert = std::max(o.cert, bits_to_double(st.cert_bits[i]));
  o.pivot = st.pivot_seg != INT_MAX;
  o.pivot_seg = st.pivot_seg;
  o.bad = o.pivot || st.bad_seg != INT_MAX || !(o.cert == o.cert);
  return o;
}

// SolveStats::reduced_ops: multiply-adds of phase 2 as a function of the
// reference plan's reduced system only (q blocks of size k; SPEC's
// "sequential fraction" law), whatever internal segmentation the GPU uses:
// speculative -- one (2H+1)-block weight product per separator;
// exact -- block-tridiagonal elimination, ~6 k^3 per block.
long long reduced_ops_of(const psg_handle* h, bool spec) {
  const long long q = h->plan.sep_count(), k = h->plan.sep_size;
  if (spec) {
    const long long H = h->generic ? (long long)blk_hb((int)k) : kHalo;
    return q * (2 * H + 1) * k * k;
  }
  return 6 * q * k * k * k;
}

void ensure_exact_generic(psg_handle* h, cudaStream_t s) {
  if (h->exact_factored) return;
  h->gen.launches = 0;
  h->gen.factor(s);
  h->exact_factored = true;
}

// The reference plan's reduced system (ReducedSystem, psg_reduced_* and
// psg_solve_reduced).  Generic handles have it on their exact path; a
// tridiagonal handle whose bodies were refined internally (bodies > 1056
// rows: its own levels carry extra separators) gets it from the generic
// exact path built on demand over the same matrix and plan.
void ensure_reduced_gen(psg_handle* h, cudaStream_t s) {
  if (h->generic) {
    ensure_exact_generic(h, s);
    return;
  }
  if (h->gen.lv.empty() || h->gen_ref_data != h->A.data) {
    SMView V{PSG_BANDED, h->A.n, 1, 1, 1, h->A.data, nullptr, 0, 0};
    CUDA_TRY(cudaStreamSynchronize(s));
    h->gen.build(V, h->plan.p);
    h->gen_ref_data = h->A.data;
    h->gen_ref_factored = false;
  }
  if (!h->gen_ref_factored) {
    h->gen.launches = 0;
    h->gen.factor(s);
    h->gen_ref_factored = true;
  }
}

// Block kinds: enqueue one speculative solve whose status lands in device
// slot `st`, copied to host slot `hst` and marked by event `done`.
int blk_enqueue(psg_handle* h, const double* df, double* dx, cudaStream_t s, DevStatus* st, DevStatus* hst,
                cudaEvent_t done, cudaEvent_t* ev) {
  // the status slot is reset by a kernel of the solve and published to the
  // pinned host slot by its last one: no copy operation in the stream
  int launches;
  if (h->use_blk()) {
    h->blk.launches = 0;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
    h->blk.spec_solve(df, dx, st, s, ev, hst);  // its first kernel resets the status slot
    launches = h->blk.launches;
  } else {
    h->chain.launches = 0;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
    h->chain.solve(df, dx, st, s, ev, hst);
    launches = h->chain.launches;
  }
  if (ev) CUDA_TRY(cudaEventRecord(ev[3], s));
  CUDA_TRY(cudaEventRecord(done, s));
  return launches;
}

void add_phase_stats(psg_handle* h, psg_stats* stats, cudaEvent_t* ev) {
  float tf = 0, t01 = 0, t12 = 0, t23 = 0;
  cudaEventElapsedTime(&tf, h->ev_f0, h->ev_f1);
  cudaEventElapsedTime(&t01, ev[0], ev[1]);
  cudaEventElapsedTime(&t12, ev[1], ev[2]);
  cudaEventElapsedTime(&t23, ev[2], ev[3]);
  stats->factor_seconds = tf * 1e-3;
  stats->phase1_seconds += t01 * 1e-3;  // accumulate like SolveStats (src/parfact.cpp:233-237)
  stats->phase2_seconds += t12 * 1e-3;
  stats->phase3_seconds += t23 * 1e-3;
}

// Generic kinds, blocking: the block speculative path when possible, else (or
// when its certificate fails) the exact generic path with residual refinement.
// Pivoting handles: solve, certify by the normwise residual, refine once.
void piv_blocking(psg_handle* h, const double* df, double* dx, cudaStream_t s, psg_stats* stats) {
  const int n = h->A.n;
  const double* f = df;
  if (h->rot) {  // the rhs of the row-rotated matrix (ParallelFactorization::row_perm)
    h->d_fperm.alloc(n);
    piv_rotate_kernel<<<148 * 8, 256, 0, s>>>(n, 1, h->rot, df, h->d_fperm.p);
    LAUNCH_CHECK();
    f = h->d_fperm.p;
  }
  PivSolver& P = *h->piv;
  P.solve(f, dx, s, stats ? h->ev : nullptr);
  int launches = P.launches + (h->rot ? 1 : 0);
  MatView v{h->A.kind, h->A.n, h->A.m, h->A.s, h->A.r, h->A.data, h->A.corner, h->A.corner_rows, h->A.corner_cols};
  h->d_r.alloc(n);
  h->d_norm.alloc(2);
  auto resid = [&]() {
    unsigned long long hb[2];
    CUDA_TRY(cudaMemsetAsync(h->d_norm.p, 0, 2 * sizeof(unsigned long long), s));
    residual_vec_kernel<<<148 * 8, 256, 0, s>>>(v, dx, f, h->d_r.p, h->d_norm.p);
    LAUNCH_CHECK();
    CUDA_TRY(cudaMemcpyAsync(hb, h->d_norm.p, sizeof hb, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const double num = bits_to_double(hb[0]), den = bits_to_double(hb[1]);
    return den > 0 ? num / den : num;
  };
  double rel = resid();
  ++launches;
  if (rel > h->refine_tol && rel == rel) {
    h->d_d.alloc(n);
    P.solve(h->d_r.p, h->d_d.p, s, nullptr);
    axpy_kernel<<<148 * 8, 256, 0, s>>>(n, h->d_d.p, dx);
    LAUNCH_CHECK();
    launches += P.launches + 2;
    rel = resid();
  }
  if (!(rel == rel)) throw Fail{PSG_E_SINGULAR_REDUCED_SYSTEM, "non-finite solution"};
  h->solve_launches = launches;
  if (stats) {
    add_phase_stats(h, stats, h->ev);
    stats->reduced_ops += P.reduced_ops();
    stats->certificate = std::max(stats->certificate, rel);
    stats->speculative = 0;
  }
}

void generic_blocking(psg_handle* h, const double* df, double* dx, cudaStream_t s, psg_stats* stats) {
  int fallbacks = 0;
  if (h->use_blk() || h->use_chain()) {
    if (!h->spec_factored) run_factor(h, s);
    const int launches = blk_enqueue(h, df, dx, s, h->d_status.p, h->h_status, h->ev_done, stats ? h->ev : nullptr);
    CUDA_TRY(cudaEventSynchronize(h->ev_done));
    const Outcome o = read_status(*h->h_status);
    if (!o.bad && o.cert <= h->cert_tol) {
      h->solve_launches = launches;
      if (stats) {
        add_phase_stats(h, stats, h->ev);
        stats->reduced_ops += reduced_ops_of(h, true);
        stats->certificate = std::max(stats->certificate, o.cert);
        stats->speculative = 1;
      }
      return;
    }
    fallbacks = 1;
    h->speculative = false;  // speculative interface rejected: this handle goes exact
  }
  ensure_exact_generic(h, s);
  double cert = 0;
  h->solve_launches = generic_solve(h, df, dx, s, stats != nullptr, &cert);
  if (stats) {
    add_phase_stats(h, stats, h->ev);
    stats->reduced_ops += reduced_ops_of(h, false);
    stats->certificate = std::max(stats->certificate, cert);
    stats->speculative = 0;
    stats->fallbacks += fallbacks;
  }
}

// Tridiagonal: enqueue one solve attempt whose status lands in device slot
// `st`, copied to host slot `hst` and marked by event `done`.
int tri_enqueue(psg_handle* h, const double* df, double* dx, cudaStream_t s, DevStatus* st, DevStatus* hst,
                cudaEvent_t done, cudaEvent_t* ev, bool spec) {
  const int n = h->A.n;
  h->tri.launches = 0;
  if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
  if (spec) {
    // the first kernel resets the status slot, the last one publishes it to hst
    h->tri.spec_solve(make_rows(df, 0, n), dx, st, s, ev, hst);
  } else {
    DevStatus init{};
    for (int i = 0; i < kCertSlots; ++i) init.cert_bits[i] = 0ull;
    init.bad_seg = INT_MAX;
    init.pivot_seg = INT_MAX;
    *hst = init;
    CUDA_TRY(cudaMemcpyAsync(st, hst, sizeof(DevStatus), cudaMemcpyHostToDevice, s));
    h->tri.exact_solve(make_rows(df, 0, n), dx, st, s, ev);
  }
  if (ev) CUDA_TRY(cudaEventRecord(ev[3], s));
  if (!spec) CUDA_TRY(cudaMemcpyAsync(hst, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaEventRecord(done, s));
  return h->tri.launches;
}

// Blocking tridiagonal solve with the speculative -> exact fallback.
void tri_solve_blocking(psg_handle* h, const double* df, double* dx, cudaStream_t s, psg_stats* stats) {
  const bool timing = stats != nullptr;
  int fallbacks = 0, launches = 0;
  bool spec_used = false;
  double cert = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const bool spec = h->use_spec();
    if (!spec && !h->exact_factored) {  // exact mode needs its factor data (levels, reduced T)
      run_factor(h, s);
      launches += h->tri.launches;
    }
    launches += tri_enqueue(h, df, dx, s, h->d_status.p, h->h_status, h->ev_done, timing ? h->ev : nullptr, spec);
    CUDA_TRY(cudaEventSynchronize(h->ev_done));
    const Outcome o = read_status(*h->h_status);
    cert = o.cert;
    if (!o.bad && cert <= h->cert_tol) {
      spec_used = spec;
      break;
    }
    if (!spec) {
      if (o.pivot)  // parallel_factor's lowest failing partition (src/parfact.cpp:61-68)
        throw Fail{PSG_E_ZERO_PIVOT, "partition " + std::to_string(partition_of_segment(h, o.pivot_seg)) +
                                         ": zero pivot in the no-pivot elimination"};
      if (o.bad) throw Fail{PSG_E_SINGULAR_REDUCED_SYSTEM, "non-finite solution: the reduced system is singular"};
      break;  // exact mode: the certificate is reported, the result kept
    }
    ++fallbacks;  // speculative interface rejected: switch this handle to the exact path
    h->speculative = false;
  }
  h->solve_launches = launches;
  if (stats) {
    float tf = 0, t01 = 0, t12 = 0, t23 = 0;
    cudaEventElapsedTime(&tf, h->ev_f0, h->ev_f1);
    cudaEventElapsedTime(&t01, h->ev[0], h->ev[1]);
    cudaEventElapsedTime(&t12, h->ev[1], h->ev[2]);
    cudaEventElapsedTime(&t23, h->ev[2], h->ev[3]);
    stats->factor_seconds = tf * 1e-3;
    stats->phase1_seconds += t01 * 1e-3;  // accumulate like SolveStats (src/parfact.cpp:233-237)
    stats->phase2_seconds += t12 * 1e-3;
    stats->phase3_seconds += t23 * 1e-3;
    stats->reduced_ops += reduced_ops_of(h, spec_used);
    stats->certificate = std::max(stats->certificate, cert);
    stats->speculative = spec_used ? 1 : 0;
    stats->fallbacks += fallbacks;
  }
}

}  // namespace

int psg_solve(const psg_handle* hc, const double* f, double* x, int on_device, void* stream, psg_stats* stats,
              char* err, size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    order_on(h, s);
    const int n = h->A.n;
    const double* df = f;
    double* dx = x;
    // host buffers, speculative tridiagonal path: chunked pipeline (x leaves
    // while f still arrives); stats requests take the phase-timed path below
    if (!on_device && !stats && !h->piv && !h->generic && h->use_spec() && h->spec_factored && n >= (1 << 22)) {
      h->d_f.alloc(n);
      h->d_x.alloc(n);
      const int nchunk = std::min(16, std::max(2, n >> 22));
      while ((int)h->host_evs.size() < 1 + 2 * nchunk) h->host_evs.push_back(event_pool().get());
      cudaStream_t ci, co;
      copy_streams(ci, co);
      h->tri.launches = 0;
      h->tri.spec_solve_host(f, x, h->d_f.p, h->d_x.p, h->d_status.p, s, ci, co, h->host_evs.data(), nchunk,
                             h->h_status);
      CUDA_TRY(cudaEventRecord(h->ev_done, s));
      CUDA_TRY(cudaEventSynchronize(h->ev_done));
      const Outcome o = read_status(*h->h_status);
      h->solve_launches = h->tri.launches;
      if (!o.bad && o.cert <= h->cert_tol) return 0;
      h->speculative = false;  // speculative interface rejected: exact re-solve of the staged f
      tri_solve_blocking(h, h->d_f.p, h->d_x.p, s, nullptr);
      CUDA_TRY(cudaMemcpyAsync(x, h->d_x.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      CUDA_TRY(cudaEventRecord(h->ev_done, s));
      return 0;
    }
    if (!on_device) {
      h->d_f.alloc(n);
      h->d_x.alloc(n);
      CUDA_TRY(cudaMemcpyAsync(h->d_f.p, f, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      df = h->d_f.p;
      dx = h->d_x.p;
    }
    if (h->piv) {
      piv_blocking(h, df, dx, s, stats);
    } else if (h->generic) {
      generic_blocking(h, df, dx, s, stats);
    } else {
      tri_solve_blocking(h, df, dx, s, stats);
    }
    if (!on_device) {
      CUDA_TRY(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    CUDA_TRY(cudaEventRecord(h->ev_done, s));
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

// ---------------------------------------------------------------------------
// time-parallel IVP trajectory (src/odeparallel.cpp:183-233)
// ---------------------------------------------------------------------------
int psg_ode_trajectory(int m, int p, int N, const double* win, const double* g, double* out, void* stream,
                       psg_stats* stats, char* err, size_t errlen) {
  try {
    if (m < 1 || m > 8) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "the GPU trajectory solve supports dimension 1..8"};
    if (p < 1 || N < 1) throw Fail{PSG_E_INVALID_INTERVAL, "p and N must be >= 1"};
    cudaStream_t s = (cudaStream_t)stream;
    const int MB = m <= 2 ? 2 : (m <= 4 ? 4 : 8);
    const long long steps = (long long)p * N, nsteps = std::max<long long>(steps, 64), nb = nsteps + 1;
    if ((long long)MB * nb > INT_MAX) throw Fail{PSG_E_TOO_LARGE_FOR_DENSE, "trajectory too long for one solve"};
    const size_t len = size_t(MB) * MB + size_t(nsteps) * 2 * MB * MB;
    DevBuf<double> dwin, dg, ddata, dcorner, df, dx, dout;
    dwin.alloc(size_t(p) * 2 * m * m);
    dg.alloc(size_t(steps + 1) * m);
    ddata.alloc(len);
    dcorner.alloc(size_t(MB) * MB);
    df.alloc(size_t(MB) * nb);
    dx.alloc(size_t(MB) * nb);
    dout.alloc(size_t(steps + 1) * m);
    CUDA_TRY(cudaMemcpyAsync(dwin.p, win, sizeof(double) * p * 2 * m * m, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(dg.p, g, sizeof(double) * (steps + 1) * m, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(dcorner.p, 0, sizeof(double) * MB * MB, s));
    const int grid = 148 * 8, tpb = 256;
    switch (MB) {
      case 2: ode_assemble_kernel<2><<<grid, tpb, 0, s>>>(m, steps, nsteps, N, dwin.p, dg.p, ddata.p, df.p); break;
      case 4: ode_assemble_kernel<4><<<grid, tpb, 0, s>>>(m, steps, nsteps, N, dwin.p, dg.p, ddata.p, df.p); break;
      default: ode_assemble_kernel<8><<<grid, tpb, 0, s>>>(m, steps, nsteps, N, dwin.p, dg.p, ddata.p, df.p); break;
    }
    LAUNCH_CHECK();
    psg_desc A{PSG_BABD, int(MB * nb), MB, MB, 0, ddata.p, len, dcorner.p, MB, MB, 1};
    const int pp = (int)std::max<long long>(2, std::min<long long>(4096, nb / 16));
    psg_handle* h = nullptr;
    int rc = psg_factor(&A, pp, PSG_LU, 0.0, stream, &h, err, errlen);
    if (rc) return rc;
    rc = psg_solve(h, df.p, dx.p, 1, stream, stats, err, errlen);
    psg_release(h);
    if (rc) return rc;
    switch (MB) {
      case 2: ode_unpad_kernel<2><<<grid, tpb, 0, s>>>(m, steps, dx.p, dout.p); break;
      case 4: ode_unpad_kernel<4><<<grid, tpb, 0, s>>>(m, steps, dx.p, dout.p); break;
      default: ode_unpad_kernel<8><<<grid, tpb, 0, s>>>(m, steps, dx.p, dout.p); break;
    }
    LAUNCH_CHECK();
    CUDA_TRY(cudaMemcpyAsync(out, dout.p, sizeof(double) * (steps + 1) * m, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

// ---------------------------------------------------------------------------
// Parareal (pr_kernels.cuh; src/parareal.cpp:56-117)
// ---------------------------------------------------------------------------
struct psg_pr {
  int device = 0, m = 0, p = 0;
  struct Side {
    int S = 0;
    DevBuf<double> T, Minv, rhs, c;
    DevBuf<int> mat;
    PrStepper view() const { return PrStepper{S, T.p, Minv.p, rhs.n ? rhs.p : nullptr, rhs.n ? c.p : nullptr, mat.p}; }
  } F, G;
  DevBuf<double> y0, in0, in1, fine, gold, norms, tmp;
  int cur = 0;  // which of in0 / in1 holds the current inits
  double* inits() { return cur ? in1.p : in0.p; }
  double* other() { return cur ? in0.p : in1.p; }
};

namespace {

void pr_side(psg_pr::Side& sd, int m, int p, int S, int nmat, const double* T, const double* M, const int* mat,
             const double* rhs) {
  if (S < 1 || nmat < 1) throw Fail{PSG_E_INVALID_PARAMETER, "propagator needs >= 1 step and >= 1 matrix"};
  sd.S = S;
  sd.T.alloc((size_t)nmat * m * m);
  sd.Minv.alloc((size_t)nmat * m * m);
  sd.mat.alloc(p);
  CUDA_TRY(cudaMemcpy(sd.T.p, T, sizeof(double) * nmat * m * m, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(sd.Minv.p, M, sizeof(double) * nmat * m * m, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(sd.mat.p, mat, sizeof(int) * p, cudaMemcpyHostToDevice));
  if (!rhs) return;  // no forcing: c = 0 (PrStepper::c null)
  sd.rhs.alloc((size_t)p * S * m);
  sd.c.alloc((size_t)p * S * m);
  CUDA_TRY(cudaMemcpy(sd.rhs.p, rhs, sizeof(double) * (size_t)p * S * m, cudaMemcpyHostToDevice));
  const long tasks = (long)p * S;
  pr_prep_kernel<<<(unsigned)((tasks + 7) / 8), 256>>>(m, p, S, sd.Minv.p, sd.mat.p, sd.rhs.p, sd.c.p);
  LAUNCH_CHECK();
}

PrArgs pr_args(psg_pr* h, int with_fine) {
  PrArgs a{};
  a.m = h->m;
  a.p = h->p;
  a.F = h->F.view();
  a.G = h->G.view();
  a.y0 = h->y0.p;
  a.old_inits = h->inits();
  a.new_inits = h->other();
  a.fine = h->fine.p;
  a.gold = h->gold.p;
  a.norms = h->norms.p;
  a.with_fine = with_fine;
  return a;
}

void pr_smem_attr() {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (done[dev & 63]) return;
  for (const void* k : {(const void*)pr_sweep_kernel, (const void*)pr_apply_kernel})
    CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PrSmem)));
  done[dev & 63] = true;
}

// one Parareal iteration (with_fine) or the initial coarse sweep; returns {update, scale}
std::pair<double, double> pr_step(psg_pr* h, int with_fine) {
  PrArgs a = pr_args(h, with_fine);
  if (with_fine && h->p > 1) {
    const int nw = (h->m + 15) / 16;
    if (nw <= 1) pr_fine_kernel<1><<<h->p - 1, 32>>>(a);
    else if (nw == 2) pr_fine_kernel<2><<<h->p - 1, 64>>>(a);
    else if (nw == 3) pr_fine_kernel<3><<<h->p - 1, 96>>>(a);
    else pr_fine_kernel<4><<<h->p - 1, 128>>>(a);
    LAUNCH_CHECK();
  }
  pr_sweep_kernel<<<1, 32, sizeof(PrSmem)>>>(a);
  LAUNCH_CHECK();
  double nb[2];
  CUDA_TRY(cudaMemcpy(nb, h->norms.p, sizeof nb, cudaMemcpyDeviceToHost));
  h->cur ^= 1;
  return {nb[0], nb[1]};
}

}  // namespace

int psg_pr_create(int m, int p, const double* y0, int Sf, int nmat_f, const double* Tf, const double* Mf,
                  const int* matf, const double* rhsf, int Sc, int nmat_c, const double* Tc, const double* Mc,
                  const int* matc, const double* rhsc, psg_pr** out, char* err, size_t errlen) {
  *out = nullptr;
  try {
    if (m < 1 || m > kPrMaxM) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "Parareal on the GPU supports dimension 1..64"};
    if (p < 1) throw Fail{PSG_E_INVALID_INTERVAL, "need at least one window"};
    pr_smem_attr();
    std::unique_ptr<psg_pr> h(new psg_pr);
    CUDA_TRY(cudaGetDevice(&h->device));
    h->m = m;
    h->p = p;
    pr_side(h->F, m, p, Sf, nmat_f, Tf, Mf, matf, rhsf);
    pr_side(h->G, m, p, Sc, nmat_c, Tc, Mc, matc, rhsc);
    h->y0.alloc(m);
    CUDA_TRY(cudaMemcpy(h->y0.p, y0, sizeof(double) * m, cudaMemcpyHostToDevice));
    for (DevBuf<double>* b : {&h->in0, &h->in1, &h->fine, &h->gold}) {
      b->alloc((size_t)p * m);
      CUDA_TRY(cudaMemset(b->p, 0, sizeof(double) * (size_t)p * m));
    }
    h->norms.alloc(2);
    h->tmp.alloc(2 * (size_t)m);
    CUDA_TRY(cudaDeviceSynchronize());
    *out = h.release();
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_pr_set_inits(psg_pr* h, const double* inits) {
  DeviceGuard dg(h->device);
  return cudaMemcpy(h->inits(), inits, sizeof(double) * (size_t)h->p * h->m, cudaMemcpyHostToDevice) == cudaSuccess
             ? 0 : 1 + PSG_E_CUDA;
}

int psg_pr_get_inits(psg_pr* h, double* inits, double* fine) {
  DeviceGuard dg(h->device);
  const size_t bytes = sizeof(double) * (size_t)h->p * h->m;
  if (inits && cudaMemcpy(inits, h->inits(), bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1 + PSG_E_CUDA;
  if (fine && h->p > 1 &&
      cudaMemcpy(fine, h->fine.p, sizeof(double) * (size_t)(h->p - 1) * h->m, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 1 + PSG_E_CUDA;
  return 0;
}

int psg_pr_coarse_sweep(psg_pr* h, char* err, size_t errlen) {
  DeviceGuard dg(h->device);
  try {
    pr_step(h, 0);
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_pr_iterate(psg_pr* h, double* update, double* scale, char* err, size_t errlen) {
  DeviceGuard dg(h->device);
  try {
    const auto [u, sc] = pr_step(h, 1);
    if (update) *update = u;
    if (scale) *scale = sc;
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_pr_solve(psg_pr* h, double tol, int max_iter, int* iterations, double* history, int* converged, char* err,
                 size_t errlen) {
  DeviceGuard dg(h->device);
  try {
    if (!(tol > 0)) throw Fail{PSG_E_INVALID_PARAMETER, "tol must be positive"};
    if (max_iter < 0) max_iter = 2 * h->p;
    pr_step(h, 0);  // initial iterate: the sequential coarse sweep
    *iterations = 0;
    *converged = 1;
    if (h->p == 1) return 0;
    for (int k = 1; k <= max_iter; ++k) {
      const auto [u, sc] = pr_step(h, 1);
      if (history) history[k - 1] = u;
      *iterations = k;
      if (u <= tol * std::max(sc, 1e-300)) return 0;  // src/parareal.cpp:104-110
    }
    *converged = 0;
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_pr_apply(psg_pr* h, int which, int i, const double* y, double* out, char* err, size_t errlen) {
  DeviceGuard dg(h->device);
  try {
    if (i < 1 || i > h->p) throw Fail{PSG_E_INDEX_OUT_OF_RANGE, "window index"};
    CUDA_TRY(cudaMemcpy(h->tmp.p, y, sizeof(double) * h->m, cudaMemcpyHostToDevice));
    pr_apply_kernel<<<1, 32, sizeof(PrSmem)>>>((which ? h->G : h->F).view(), h->m, i, h->tmp.p, h->tmp.p + h->m);
    LAUNCH_CHECK();
    CUDA_TRY(cudaMemcpy(out, h->tmp.p + h->m, sizeof(double) * h->m, cudaMemcpyDeviceToHost));
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

void psg_pr_release(psg_pr* h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  cudaDeviceSynchronize();
  delete h;
}

namespace {

// Drain the pending asynchronous solves in order; a solve whose certificate
// failed is repaired by the exact path (the handle switches to exact mode).
void drain(psg_handle* h, psg_stats* stats) {
  std::vector<psg_handle::Pending> todo;
  todo.swap(h->pending);
  for (const auto& pd : todo) {
    CUDA_TRY(cudaEventSynchronize(h->ring_done[pd.slot]));
    const Outcome o = read_status(h->h_ring[pd.slot]);
    if (stats) {
      if (pd.timing) {  // phase times only for solves enqueued with timing
        float t01 = 0, t23 = 0;
        cudaEventElapsedTime(&t01, h->ring_t[pd.slot][0], h->ring_t[pd.slot][1]);
        cudaEventElapsedTime(&t23, h->ring_t[pd.slot][2], h->ring_t[pd.slot][3]);
        stats->phase1_seconds += t01 * 1e-3;
        stats->phase3_seconds += t23 * 1e-3;
      }
      stats->reduced_ops += reduced_ops_of(h, pd.spec);
      stats->certificate = std::max(stats->certificate, o.cert);
      stats->speculative = pd.spec ? 1 : 0;
    }
    if (!o.bad && o.cert <= h->cert_tol) continue;
    if (stats) stats->fallbacks += 1;
    h->speculative = false;
    if (h->generic)
      generic_blocking(h, pd.f, pd.x, pd.s, nullptr);
    else
      tri_solve_blocking(h, pd.f, pd.x, pd.s, nullptr);  // exact (throws on a genuine zero pivot)
  }
}

}  // namespace

int psg_solve_async(const psg_handle* hc, const double* f, double* x, int timing, void* stream, char* err,
                    size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    order_on(h, s);
    if (h->piv) {  // pivoting handles certify by a residual pass: blocking
      piv_blocking(h, f, x, s, nullptr);
      CUDA_TRY(cudaEventRecord(h->ev_done, s));
      return 0;
    }
    if (h->generic && !h->spec_mode()) {  // the exact generic path certifies by a residual pass: blocking
      generic_blocking(h, f, x, s, nullptr);
      CUDA_TRY(cudaEventRecord(h->ev_done, s));
      return 0;
    }
    if (!h->h_ring) {
      CUDA_TRY(cudaMallocHost(&h->h_ring, sizeof(DevStatus) * psg_handle::kRing));
      h->d_ring.alloc(psg_handle::kRing);
      for (int i = 0; i < psg_handle::kRing; ++i) {
        h->ring_done[i] = event_pool().get();
        for (int j = 0; j < 4; ++j) h->ring_t[i][j] = event_pool().get();
      }
    }
    if ((int)h->pending.size() >= psg_handle::kRing) drain(h, nullptr);
    const int slot = (int)(h->async_count++ % psg_handle::kRing);
    const bool spec = h->spec_mode();
    const int launches =
        h->generic ? blk_enqueue(h, f, x, s, h->d_ring.p + slot, h->h_ring + slot, h->ring_done[slot],
                                 timing ? h->ring_t[slot] : nullptr)
                   : tri_enqueue(h, f, x, s, h->d_ring.p + slot, h->h_ring + slot, h->ring_done[slot],
                                 timing ? h->ring_t[slot] : nullptr, spec);
    h->pending.push_back(psg_handle::Pending{slot, f, x, s, spec, timing != 0, launches});
    h->solve_launches = launches;
    CUDA_TRY(cudaEventRecord(h->ev_done, s));
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_sync(const psg_handle* hc, psg_stats* stats, char* err, size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    if (stats) {
      float tf = 0;
      CUDA_TRY(cudaEventSynchronize(h->ev_f1));
      cudaEventElapsedTime(&tf, h->ev_f0, h->ev_f1);
      stats->factor_seconds = tf * 1e-3;
    }
    drain(h, stats);
    if (h->has_carried) {  // solves drained early by psg_refactor
      if (stats) {
        stats->phase1_seconds += h->carried.phase1_seconds;
        stats->phase3_seconds += h->carried.phase3_seconds;
        stats->reduced_ops += h->carried.reduced_ops;
        stats->certificate = std::max(stats->certificate, h->carried.certificate);
        stats->fallbacks += h->carried.fallbacks;
      }
      h->carried = psg_stats{};
      h->has_carried = false;
    }
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

// New matrix values with the same structure (kind, n, m, s, r, corner shape):
// recompute the factor data on the handle's buffers (no re-planning).
int psg_refactor(psg_handle* h, const psg_desc* A, void* stream, char* err, size_t errlen) {
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    validate(*A);
    const int hs = h->A.s - h->rot, hr = h->rot ? h->rot : h->A.r;  // bandwidths as given (before permute_corner)
    if (A->kind != h->A.kind || A->n != h->A.n || A->m != h->A.m || A->s != hs || A->r != hr ||
        A->corner_rows != h->A.corner_rows || A->corner_cols != h->A.corner_cols)
      throw Fail{PSG_E_DIMENSION_MISMATCH, "psg_refactor needs the factored structure"};
    cudaStream_t s = (cudaStream_t)stream;
    order_on(h, s);
    // Pending asynchronous solves were enqueued against the current matrix.
    // When the new values arrive in another buffer (or through the handle's
    // own copy of a host matrix) the old values are about to become
    // unreachable, so those solves are drained -- a failed certificate is
    // repaired against the matrix it was enqueued for -- before anything is
    // replaced; their statistics are reported at the next psg_sync.  A
    // refactor on the same device buffer keeps them pending (stream order
    // runs them on the old factor data; psg.h: psg_sync before overwriting A
    // in place).
    if (!h->pending.empty() &&
        (!A->on_device || A->data != h->A.data || A->corner != h->A.corner || h->piv)) {
      drain(h, &h->carried);
      h->has_carried = true;
    }
    if (h->piv) {  // new values may defer other pivots: the reduced layout is rebuilt
      CUDA_TRY(cudaEventSynchronize(h->ev_done));
      piv_set_matrix(h, *A, s);
      CUDA_TRY(cudaStreamSynchronize(s));
      h->piv->A.data = h->A.data;
      h->piv->A.corner = h->A.corner;
      run_factor(h, s);
      CUDA_TRY(cudaEventRecord(h->ev_done, s));
      return 0;
    }
    const double* data = A->data;
    const double* corner = A->corner;
    if (!A->on_device) {
      h->own_data.alloc(A->data_len);
      CUDA_TRY(cudaMemcpyAsync(h->own_data.p, A->data, sizeof(double) * A->data_len, cudaMemcpyHostToDevice, s));
      data = h->own_data.p;
      if (A->corner) {
        const size_t cn = (size_t)A->corner_rows * A->corner_cols;
        h->own_corner.alloc(cn);
        CUDA_TRY(cudaMemcpyAsync(h->own_corner.p, A->corner, sizeof(double) * cn, cudaMemcpyHostToDevice, s));
        corner = h->own_corner.p;
      }
    }
    const bool moved = data != h->A.data || corner != h->A.corner;
    h->A.data = data;
    h->A.corner = corner;
    if (h->generic) {
      if (moved) {
        SMView V{h->A.kind, h->A.n, h->A.m, h->A.s, h->A.r, h->A.data, h->A.corner, h->A.corner_rows,
                 h->A.corner_cols};
        CUDA_TRY(cudaStreamSynchronize(s));
        h->gen.build(V, h->plan.p);
        h->blk.set_data(h->A.data);
        h->chain.set_data(h->A.data, h->A.corner);
      }
    } else if (moved) {
      h->tri.A0 = tri_rows(h->A);
      if (!h->tri.lv.empty()) h->tri.lv[0]->A = h->tri.A0;
    }
    h->spec_factored = h->exact_factored = false;
    h->gen_ref_factored = false;
    h->speculative = true;  // a new matrix gets a fresh speculation
    run_factor(h, s);
    CUDA_TRY(cudaEventRecord(h->ev_done, s));
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_reduced_info(const psg_handle* h, int* q, int* dim, int* k, int* has_corner) {
  if (h->piv) {
    if (q) *q = h->piv->q;
    if (dim) *dim = h->piv->dim;
    if (k) *k = h->plan.sep_size;
    if (has_corner) *has_corner = h->plan.has_corner ? 1 : 0;
    return 0;
  }
  const int qq = h->plan.sep_count();
  if (q) *q = qq;
  if (dim) *dim = qq * h->plan.sep_size;
  if (k) *k = h->plan.sep_size;
  if (has_corner) *has_corner = h->plan.has_corner ? 1 : 0;
  return 0;
}

int psg_reduced_layout(const psg_handle* h, int* positions, int* sizes) {
  if (h->piv) {
    for (int j = 0; j < h->piv->q; ++j) {
      if (positions) positions[j] = h->piv->rpos[j];
      if (sizes) sizes[j] = h->piv->rsize[j];
    }
    return 0;
  }
  for (int j = 0; j < h->plan.sep_count(); ++j) {
    if (positions) positions[j] = h->plan.sep_start(j);
    if (sizes) sizes[j] = h->plan.sep_size;
  }
  return 0;
}

int psg_reduced_dense(const psg_handle* hc, double* T, char* err, size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  try {
    {
      std::lock_guard<std::mutex> g(h->mu);
      CUDA_TRY(cudaEventSynchronize(h->ev_done));
      if (h->piv) {
        h->piv->dense_T(T);
        return 0;
      }
    }
    const int q = h->plan.sep_count(), k = h->plan.sep_size, kk = k * k, dim = q * k;
    std::vector<double> dg_(static_cast<size_t>(q) * kk), sb(static_cast<size_t>(q) * kk), sp(static_cast<size_t>(q) * kk);
    const int rc = psg_reduced_blocks(hc, dg_.data(), sb.data(), sp.data(), err, errlen);
    if (rc) return rc;
    std::fill(T, T + (size_t)dim * dim, 0.0);
    for (int j = 0; j < q; ++j)
      for (int t = 0; t < k; ++t)
        for (int u = 0; u < k; ++u) {
          T[(size_t)(j * k + t) * dim + j * k + u] = dg_[(size_t)j * kk + t * k + u];
          if (j > 0) T[(size_t)(j * k + t) * dim + (j - 1) * k + u] = sb[(size_t)j * kk + t * k + u];
          if (j + 1 < q) T[(size_t)(j * k + t) * dim + (j + 1) * k + u] = sp[(size_t)j * kk + t * k + u];
        }
    if (h->plan.has_corner)
      for (int t = 0; t < k; ++t)
        for (int u = 0; u < k; ++u) T[(size_t)t * dim + (q - 1) * k + u] += sb[t * k + u];
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_reduced_blocks(const psg_handle* hc, double* diag, double* sub, double* super, char* err, size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    CUDA_TRY(cudaEventSynchronize(h->ev_done));
    if (h->piv) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "reduced system has adaptive extras: use psg_reduced_dense"};
    if (h->generic || h->refined) {  // parallel_factor's ReducedSystem comes from the exact path
      ensure_reduced_gen(h, nullptr);
      CUDA_TRY(cudaDeviceSynchronize());
      GenLevel& L = *h->gen.lv[0];
      const int q = L.q, k = L.k, kk = k * k;
      std::vector<double> T(L.Tdata.n), C(kk, 0.0);
      CUDA_TRY(cudaMemcpy(T.data(), L.Tdata.p, sizeof(double) * T.size(), cudaMemcpyDeviceToHost));
      if (L.corner) CUDA_TRY(cudaMemcpy(C.data(), L.Tcorner.p, sizeof(double) * kk, cudaMemcpyDeviceToHost));
      auto put = [&](double* dst, int j, const double* src, int pitch) {
        if (!dst) return;
        for (int t = 0; t < k; ++t)
          for (int u = 0; u < k; ++u) dst[(long)j * kk + t * k + u] = src ? src[(long)t * pitch + u] : 0.0;
      };
      for (int j = 0; j < q; ++j) {
        if (!L.corner) {
          const long off = j == 0 ? 0 : (3L * j - 1) * kk;
          const int dblk = j > 0 ? 1 : 0;
          put(sub, j, j > 0 ? &T[off] : nullptr, k);
          put(diag, j, &T[off + (long)dblk * kk], k);
          put(super, j, j < q - 1 ? &T[off + (long)(dblk + 1) * kk] : nullptr, k);
        } else {
          const long off = j == 0 ? 0 : (long)k * 2 * k + (long)(j - 1) * k * 3 * k;
          const int width = (j == 0 || j == q - 1) ? 2 * k : 3 * k;
          const double* row = &T[off];
          if (j == 0) {
            put(sub, 0, C.data(), k);  // sub[0] carries the corner coupling (psg.h)
            put(diag, 0, row, width);
            put(super, 0, q > 1 ? row + k : nullptr, width);
          } else {
            put(sub, j, row, width);
            put(diag, j, row + k, width);
            put(super, j, j < q - 1 ? row + 2 * k : nullptr, width);
          }
        }
      }
      return 0;
    }
    const int ns = h->tri.S0.nseg - 1;
    if (h->use_spec() && h->spec_factored) {
      // speculative reduced matrix: diagonal (beta = gamma = 0 below rho^L)
      h->tri.spec_tdiag(nullptr);
      CUDA_TRY(cudaDeviceSynchronize());
      if (diag) CUDA_TRY(cudaMemcpy(diag, h->tri.Tdiag.p, sizeof(double) * ns, cudaMemcpyDeviceToHost));
      if (sub) std::fill(sub, sub + ns, 0.0);
      if (super) std::fill(super, super + ns, 0.0);
      return 0;
    }
    TriLevel& L = *h->tri.lv[0];
    if (diag) CUDA_TRY(cudaMemcpy(diag, L.Tdiag.p, sizeof(double) * ns, cudaMemcpyDeviceToHost));
    if (sub) CUDA_TRY(cudaMemcpy(sub, L.Tsub.p, sizeof(double) * ns, cudaMemcpyDeviceToHost));
    if (super) CUDA_TRY(cudaMemcpy(super, L.Tsup.p, sizeof(double) * ns, cudaMemcpyDeviceToHost));
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_solve_reduced(const psg_handle* hc, const double* rhs, double* x, int on_device, void* stream,
                      psg_stats* stats, char* err, size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    order_on(h, s);
    if (h->piv) {
      const int dim = h->piv->dim;
      DevBuf<double> dr, dxv;
      const double* r = rhs;
      double* xo = x;
      if (!on_device) {
        dr.alloc(dim);
        dxv.alloc(dim);
        CUDA_TRY(cudaMemcpyAsync(dr.p, rhs, sizeof(double) * dim, cudaMemcpyHostToDevice, s));
        r = dr.p;
        xo = dxv.p;
      }
      h->piv->solve_reduced(r, xo, s);
      if (!on_device) CUDA_TRY(cudaMemcpyAsync(x, xo, sizeof(double) * dim, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      CUDA_TRY(cudaEventRecord(h->ev_done, s));
      if (stats) stats->reduced_ops += h->piv->reduced_ops();
      return 0;
    }
    if (h->generic || h->refined) {
      ensure_reduced_gen(h, s);
      if (h->gen.lv.size() < 2) throw Fail{PSG_E_INVALID_PARAMETER, "no reduced system"};
      const int dim = h->gen.lv[0]->q * h->gen.lv[0]->k;
      DevBuf<double> dr, dxv;
      const double* r = rhs;
      double* xo = x;
      if (!on_device) {
        dr.alloc(dim);
        dxv.alloc(dim);
        CUDA_TRY(cudaMemcpyAsync(dr.p, rhs, sizeof(double) * dim, cudaMemcpyHostToDevice, s));
        r = dr.p;
        xo = dxv.p;
      }
      h->gen.solve(r, xo, nullptr, s, nullptr, 1);
      h->gen.restore_level1_wiring();
      if (!on_device) CUDA_TRY(cudaMemcpyAsync(x, xo, sizeof(double) * dim, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      CUDA_TRY(cudaEventRecord(h->ev_done, s));
      if (stats) stats->reduced_ops += reduced_ops_of(h, false);
      return 0;
    }
    if (!h->exact_factored) {  // the exact reduced matrix T (parallel_factor's ReducedSystem)
      h->tri.launches = 0;
      h->tri.exact_factor(s);
      h->exact_factored = true;
    }
    const int q = h->tri.S0.nseg - 1;
    DevBuf<double> dr, dxv;
    const double* r = rhs;
    double* xo = x;
    if (!on_device) {
      dr.alloc(q);
      dxv.alloc(q);
      CUDA_TRY(cudaMemcpyAsync(dr.p, rhs, sizeof(double) * q, cudaMemcpyHostToDevice, s));
      r = dr.p;
      xo = dxv.p;
    }
    h->tri.exact_solve(make_rows(r, 0, q), xo, nullptr, s, nullptr, 1);
    h->tri.restore_level1_wiring();
    if (!on_device) CUDA_TRY(cudaMemcpyAsync(x, xo, sizeof(double) * q, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaEventRecord(h->ev_done, s));
    if (stats) stats->reduced_ops += reduced_ops_of(h, false);
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_reduced_rhs(const psg_handle* hc, const double* f, double* out, int on_device, void* stream, char* err,
                    size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    order_on(h, s);
    if (h->piv) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "reduced rhs of a pivoting factorization: use solve"};
    if (h->rot) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "reduced rhs of a row-rotated (circulant) system"};
    const int n = h->A.n;
    const double* df = f;
    DevBuf<double> dfb, dob;
    if (!on_device) {
      dfb.alloc(n);
      CUDA_TRY(cudaMemcpyAsync(dfb.p, f, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      df = dfb.p;
    }
    const double* rr = nullptr;
    size_t dim = 0;
    if (h->generic || h->refined) {
      ensure_reduced_gen(h, s);
      if (h->gen.lv.size() < 2) throw Fail{PSG_E_INVALID_PARAMETER, "no reduced system"};
      rr = h->gen.condense(df, s);
      dim = (size_t)h->gen.lv[0]->q * h->gen.lv[0]->k;
    } else {
      if (!h->exact_factored) {
        h->tri.launches = 0;
        h->tri.exact_factor(s);
        h->exact_factored = true;
      }
      rr = h->tri.exact_condense(make_rows(df, 0, n), s);
      dim = (size_t)h->tri.S0.nseg - 1;
    }
    CUDA_TRY(cudaMemcpyAsync(out, rr, sizeof(double) * dim, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                             s));
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaEventRecord(h->ev_done, s));
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

// Debug/inspection: copy an internal buffer to the host.  what = 0: speculative
// weight rows (nsep x 68), 1: speculative Tdiag (nsep).  Returns the count.
long psg_debug_buffer(const psg_handle* hc, int what, double* out, long cap) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  DeviceGuard dg(h->device);
  std::lock_guard<std::mutex> g(h->mu);
  if (cudaEventSynchronize(h->ev_done) != cudaSuccess) return -1;
  if (what != 1) return -1;  // the separator weights are no longer formed (tri_spec_fused_kernel)
  if (h->use_spec() && h->spec_factored) {
    try {
      h->tri.spec_tdiag(nullptr);
    } catch (const Fail&) {
      return -1;
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  }
  const DevBuf<double>& b = h->tri.Tdiag;
  const long nsep = h->tri.S0.nseg - 1;
  const long cnt = nsep;
  if (!b.p || cnt > cap) return -cnt;
  if (cudaMemcpy(out, b.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return cnt;
}

int psg_validate(const psg_desc* A, char* err, size_t errlen) {
  try {
    validate(*A);
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

size_t psg_body_entry_count(int kind, int n, int m, int s, int r) { return body_entry_count(kind, n, m, s, r); }

int psg_matvec(const psg_desc* A, const double* x, double* y, int on_device, void* stream, char* err, size_t errlen) {
  try {
    validate(*A);
    cudaStream_t s = (cudaStream_t)stream;
    MatView v{A->kind, A->n, A->m, A->s, A->r, A->data, A->corner, A->corner_rows, A->corner_cols};
    DevBuf<double> dd, dc, dxv, dyv;
    if (!A->on_device) {
      dd.alloc(A->data_len);
      CUDA_TRY(cudaMemcpyAsync(dd.p, A->data, sizeof(double) * A->data_len, cudaMemcpyHostToDevice, s));
      v.data = dd.p;
      if (A->corner) {
        const size_t cn = (size_t)A->corner_rows * A->corner_cols;
        dc.alloc(cn);
        CUDA_TRY(cudaMemcpyAsync(dc.p, A->corner, sizeof(double) * cn, cudaMemcpyHostToDevice, s));
        v.corner = dc.p;
      }
    }
    const double* xd = x;
    double* yd = y;
    if (!on_device) {
      dxv.alloc(A->n);
      dyv.alloc(A->n);
      CUDA_TRY(cudaMemcpyAsync(dxv.p, x, sizeof(double) * A->n, cudaMemcpyHostToDevice, s));
      xd = dxv.p;
      yd = dyv.p;
    }
    matvec_kernel<<<148 * 8, 256, 0, s>>>(v, xd, yd);
    LAUNCH_CHECK();
    if (!on_device) CUDA_TRY(cudaMemcpyAsync(y, yd, sizeof(double) * A->n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_residual(const psg_desc* A, const double* x, const double* f, int on_device, void* stream, double* out,
                 char* err, size_t errlen) {
  try {
    validate(*A);
    cudaStream_t s = (cudaStream_t)stream;
    DevBuf<double> dd, dc, dxv, dfv;
    MatView v{A->kind, A->n, A->m, A->s, A->r, A->data, A->corner, A->corner_rows, A->corner_cols};
    if (!A->on_device) {
      dd.alloc(A->data_len);
      CUDA_TRY(cudaMemcpyAsync(dd.p, A->data, sizeof(double) * A->data_len, cudaMemcpyHostToDevice, s));
      v.data = dd.p;
      if (A->corner) {
        const size_t cn = (size_t)A->corner_rows * A->corner_cols;
        dc.alloc(cn);
        CUDA_TRY(cudaMemcpyAsync(dc.p, A->corner, sizeof(double) * cn, cudaMemcpyHostToDevice, s));
        v.corner = dc.p;
      }
    }
    const double* xd = x;
    const double* fd = f;
    if (!on_device) {
      dxv.alloc(A->n);
      dfv.alloc(A->n);
      CUDA_TRY(cudaMemcpyAsync(dxv.p, x, sizeof(double) * A->n, cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(dfv.p, f, sizeof(double) * A->n, cudaMemcpyHostToDevice, s));
      xd = dxv.p;
      fd = dfv.p;
    }
    DevBuf<unsigned long long> o;
    o.alloc(2);
    CUDA_TRY(cudaMemsetAsync(o.p, 0, 2 * sizeof(unsigned long long), s));
    residual_kernel<<<148 * 8, 256, 0, s>>>(v, xd, fd, o.p);
    LAUNCH_CHECK();
    unsigned long long hb[2];
    CUDA_TRY(cudaMemcpyAsync(hb, o.p, sizeof hb, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const double num = bits_to_double(hb[0]);
    const double den = bits_to_double(hb[1]);
    *out = den > 0 ? num / den : num;
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

}  // extern "C"

#ifdef PSG_PROF
// chain_solve_kernel phase stamps (a -DPSG_PROF build only; tools/prof_cs.py)
extern "C" int psg_prof_dump(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, psg::g_prof, sizeof(long long) * 2 * 1024 * 6);
}
// per-kernel timeline stamps (tools/tl_probe.py): out = 16 x 4 words; reset re-arms the minima / maxima
extern "C" int psg_tl_dump(unsigned long long* out, int reset) {
  const int rc = (int)cudaMemcpyFromSymbol(out, psg::g_tl, sizeof(unsigned long long) * 64);
  if (reset) {
    unsigned long long init[64];
    for (int k = 0; k < 16; ++k) {
      init[4 * k] = ~0ull;  // TL_MIN slots: [id][0] and, for the passes, [id][2]
      init[4 * k + 1] = 0;
      init[4 * k + 2] = (k == 2 || k == 4) ? ~0ull : 0;
      init[4 * k + 3] = 0;
    }
    for (int k = 6; k < 16; ++k) init[4 * k] = 0;  // TL_MAX only
    cudaMemcpyToSymbol(psg::g_tl, init, sizeof(init));
  }
  return rc;
}
#endif
