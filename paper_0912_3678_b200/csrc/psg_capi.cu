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
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/psg.h"
#include "gen_kernels.cuh"
#include "psg_common.cuh"
#include "tri_kernels.cuh"

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

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    reset();
    CUDA_TRY(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
    n = count;
  }
};

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
// partition plan: plan_partition (src/partition.cpp:52-105)
// ----------------------------------------------------------------------------
struct Plan {
  int kind = 0, n = 0, m = 1, p = 0, sep_size = 0;
  bool has_corner = false;
  std::vector<int> body_begin, body_end, sep_start;
};

Plan make_plan(const psg_desc& A, int p) {
  if (p < 2) throw Fail{PSG_E_TOO_MANY_PARTITIONS, "p must be >= 2"};
  if (A.kind == PSG_CIRCULANT) throw Fail{PSG_E_UNSUPPORTED_KIND, "circulant-like matrices are not supported on the GPU path"};
  Plan P;
  P.kind = A.kind;
  P.n = A.n;
  P.m = A.m;
  P.p = p;
  P.sep_size = A.kind == PSG_BANDED ? std::max(A.s, A.r) : A.m;
  P.has_corner = A.kind == PSG_BABD;
  const int k = P.sep_size;
  const long seps = P.has_corner ? p + 1L : p - 1L;
  const int unit = A.kind == PSG_BANDED ? 1 : A.m;
  if (k % unit != 0) throw Fail{PSG_E_UNSUPPORTED_KIND, "separator does not tile blocks"};
  const long n_units = A.n / unit, k_units = k / unit;
  const long body_total = n_units - seps * k_units;
  const long min_body = std::max(1L, k_units);
  if (body_total < (long)p * min_body)
    throw Fail{PSG_E_TOO_MANY_PARTITIONS, "n too small for p = " + std::to_string(p) + " partitions of this kind"};
  const long base = body_total / p, rem = body_total % p;
  P.body_begin.resize(p);
  P.body_end.resize(p);
  long cursor = 0;
  if (P.has_corner) {
    P.sep_start.push_back(int(cursor * unit));
    cursor += k_units;
  }
  for (int i = 0; i < p; ++i) {
    const long units = base + (i < rem ? 1 : 0);
    P.body_begin[i] = int(cursor * unit);
    P.body_end[i] = int((cursor + units) * unit);
    cursor += units;
    if (i < p - 1 || P.has_corner) {
      P.sep_start.push_back(int(cursor * unit));
      cursor += k_units;
    }
  }
  return P;
}

// ----------------------------------------------------------------------------
// Tridiagonal multi-level partition solver
// ----------------------------------------------------------------------------
constexpr int kNT = 64;
constexpr int kMaxSeg = 17 * kNT;  // 1088 rows per segment (one CTA)

struct TriLevel {
  TriRows A{};
  RowArr F{};
  double* x = nullptr;  // output of this level (rows of this level's system)
  int q = 0;            // rows
  int nseg = 0, maxlen = 0;
  std::vector<int> h_start, h_len;
  DevBuf<int> start, len;
  DevBuf<double> mat, rhsv;                       // 4*nseg, 2*nseg
  DevBuf<double> Tsub, Tdiag, Tsup, rhs_next, x_next;  // nseg-1
  DevBuf<double2> partR, partL;
  DevBuf<int> counters;
};

// Split q rows into segments of <= kMaxSeg rows separated by single rows,
// following the reference plan formula (equal bodies, remainder first).
void segment_uniform(int q, std::vector<int>& st, std::vector<int>& ln) {
  st.clear();
  ln.clear();
  if (q <= kMaxSeg) {
    st.push_back(0);
    ln.push_back(q);
    return;
  }
  const int p = (q + 1 + 1023) / 1024;  // ~1023-row bodies
  const long body_total = (long)q - (p - 1);
  const long base = body_total / p, rem = body_total % p;
  long cursor = 0;
  for (int i = 0; i < p; ++i) {
    const long u = base + (i < rem ? 1 : 0);
    st.push_back(int(cursor));
    ln.push_back(int(u));
    cursor += u + 1;
  }
}

template <int M>
void launch_segment_solve(const TriSolveArgs& a, int nseg, cudaStream_t s) {
  constexpr int bytes = TriSmem<M, kNT>::BYTES;
  tri_segment_solve_kernel<M, kNT><<<nseg, kNT, bytes, s>>>(a);
}

void segment_solve(const TriSolveArgs& a, int nseg, int maxlen, cudaStream_t s) {
  if (maxlen <= 3 * kNT)
    launch_segment_solve<3>(a, nseg, s);
  else if (maxlen <= 5 * kNT)
    launch_segment_solve<5>(a, nseg, s);
  else if (maxlen <= 9 * kNT)
    launch_segment_solve<9>(a, nseg, s);
  else if (maxlen <= 17 * kNT)
    launch_segment_solve<17>(a, nseg, s);
  else
    throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "segment longer than the per-CTA capacity"};
  LAUNCH_CHECK();
}

struct TriSolver {
  std::vector<std::unique_ptr<TriLevel>> lv;
  int launches = 0;

  // Level 0 = the user's matrix segmented by the (refined) plan.
  void build(const TriRows& A0, int n, const std::vector<int>& st, const std::vector<int>& ln) {
    lv.clear();
    auto L0 = std::make_unique<TriLevel>();
    L0->A = A0;
    L0->q = n;
    L0->h_start = st;
    L0->h_len = ln;
    lv.push_back(std::move(L0));
    for (;;) {
      TriLevel& L = *lv.back();
      L.nseg = (int)L.h_start.size();
      L.maxlen = *std::max_element(L.h_len.begin(), L.h_len.end());
      L.start.alloc(L.nseg);
      L.len.alloc(L.nseg);
      CUDA_TRY(cudaMemcpy(L.start.p, L.h_start.data(), sizeof(int) * L.nseg, cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(L.len.p, L.h_len.data(), sizeof(int) * L.nseg, cudaMemcpyHostToDevice));
      if (L.nseg == 1) break;
      const int ns = L.nseg - 1;
      L.mat.alloc(4 * (size_t)L.nseg);
      L.rhsv.alloc(2 * (size_t)L.nseg);
      L.Tsub.alloc(ns);
      L.Tdiag.alloc(ns);
      L.Tsup.alloc(ns);
      L.rhs_next.alloc(ns);
      L.x_next.alloc(ns);
      if (lv.size() == 1) {
        L.partR.alloc(ns);
        L.partL.alloc(ns);
        L.counters.alloc(ns);
        CUDA_TRY(cudaMemset(L.counters.p, 0, sizeof(int) * ns));
      }
      auto N = std::make_unique<TriLevel>();
      N->A.a = RowArr{L.Tsub.p, 1, ns};
      N->A.b = RowArr{L.Tdiag.p, 0, ns};
      N->A.c = RowArr{L.Tsup.p, 0, ns - 1};
      N->F = RowArr{L.rhs_next.p, 0, ns};
      N->x = L.x_next.p;
      N->q = ns;
      segment_uniform(ns, N->h_start, N->h_len);
      lv.push_back(std::move(N));
    }
  }

  static int blocks(long work, int tpb) { return (int)((work + tpb - 1) / tpb); }

  void factor(int H, cudaStream_t s) {
    for (size_t l = 0; l + 1 < lv.size(); ++l) {
      TriLevel& L = *lv[l];
      tri_interface_kernel<true, false><<<blocks(2L * L.nseg, 128), 128, 0, s>>>(
          L.A, RowArr{nullptr, 0, 0}, L.start.p, L.len.p, L.nseg, H, L.mat.p, nullptr);
      LAUNCH_CHECK();
      tri_assemble_matrix_kernel<<<blocks(L.nseg - 1, 256), 256, 0, s>>>(L.A, L.start.p, L.len.p, L.nseg - 1,
                                                                         L.mat.p, L.Tsub.p, L.Tdiag.p, L.Tsup.p);
      LAUNCH_CHECK();
      launches += 2;
    }
  }

  // phase1: condense + rhs assembly down the levels; phase2: deepest direct
  // solve + upper-level back-substitutions; phase3: level-0 back-substitution.
  void solve(const RowArr& F0, double* x0, int H, DevStatus* st, cudaStream_t s, cudaEvent_t* ev, int from = 0) {
    lv[from]->F = F0;
    lv[from]->x = x0;
    for (size_t l = from; l + 1 < lv.size(); ++l) {
      TriLevel& L = *lv[l];
      tri_interface_kernel<false, true><<<blocks(2L * L.nseg, 128), 128, 0, s>>>(
          L.A, L.F, L.start.p, L.len.p, L.nseg, H, nullptr, L.rhsv.p);
      LAUNCH_CHECK();
      tri_assemble_rhs_kernel<<<blocks(L.nseg - 1, 256), 256, 0, s>>>(L.A, L.F, L.start.p, L.len.p, L.nseg - 1,
                                                                      L.rhsv.p, L.rhs_next.p);
      LAUNCH_CHECK();
      launches += 2;
      if (l == (size_t)from && ev) cudaEventRecord(ev[1], s);
    }
    for (size_t l = lv.size(); l-- > (size_t)from;) {
      TriLevel& L = *lv[l];
      if (l == (size_t)from && ev && lv.size() > (size_t)from + 1) cudaEventRecord(ev[2], s);
      TriSolveArgs a{};
      a.A = L.A;
      a.F = L.F;
      a.seg_start = L.start.p;
      a.seg_len = L.len.p;
      a.nseg = L.nseg;
      a.xsep = L.nseg > 1 ? L.x_next.p : nullptr;
      a.x = L.x;
      a.status = st;
      if (l == 0 && L.nseg > 1) {
        a.partR = L.partR.p;
        a.partL = L.partL.p;
        a.counters = L.counters.p;
      }
      segment_solve(a, L.nseg, L.maxlen, s);
      launches += 1;
    }
  }

  long long reduced_ops() const {
    long long ops = 0;
    for (size_t l = 1; l < lv.size(); ++l) ops += 12LL * lv[l]->q;
    return ops;
  }
};

}  // namespace

// ----------------------------------------------------------------------------
// the handle
// ----------------------------------------------------------------------------
struct psg_handle {
  psg_desc A{};  // device view
  Plan plan;
  int strategy = 0;
  DevBuf<double> own_data, own_corner;
  TriSolver tri;
  std::vector<int> seg_start, seg_len;  // level-0 segmentation (refined plan)
  bool refined = false;
  // options
  bool speculative = true;
  int halo = 32;
  double cert_tol = 1e-14;
  // state
  bool factored_exact = false;  // factor data computed in exact mode
  DevBuf<DevStatus> d_status;
  DevStatus* h_status = nullptr;  // pinned
  DevBuf<double> d_f, d_x;        // host-path staging
  std::mutex mu;
  int factor_launches = 0, solve_launches = 0;
  double factor_seconds = 0;
  ~psg_handle() {
    if (h_status) cudaFreeHost(h_status);
  }
};

namespace {

TriRows tri_rows(const psg_desc& A) {
  const double* d = A.data;
  const int n = A.n;
  return TriRows{RowArr{d - 1, 1, n}, RowArr{d + (n - 1), 0, n}, RowArr{d + (2L * n - 1), 0, n - 1}};
}

void refine_segments(const Plan& P, std::vector<int>& st, std::vector<int>& ln, bool& refined) {
  st.clear();
  ln.clear();
  refined = false;
  for (int i = 0; i < P.p; ++i) {
    const int b = P.body_begin[i], L = P.body_end[i] - b;
    if (L <= kMaxSeg) {
      st.push_back(b);
      ln.push_back(L);
      continue;
    }
    refined = true;
    const int t = (L + 1 + kMaxSeg) / (kMaxSeg + 1);  // sub-bodies
    const long body = (long)L - (t - 1);
    const long base = body / t, rem = body % t;
    long cur = b;
    for (int u = 0; u < t; ++u) {
      const long len = base + (u < rem ? 1 : 0);
      st.push_back(int(cur));
      ln.push_back(int(len));
      cur += len + 1;
    }
  }
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
    case PSG_QR: throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "pivoting strategies have no GPU path"};
    default: throw Fail{PSG_E_INVALID_PARAMETER, "unknown strategy"};
  }
}

bool is_tridiag(const psg_desc& A) { return A.kind == PSG_BANDED && A.s == 1 && A.r == 1; }

void run_factor(psg_handle* h, cudaStream_t s) {
  const int H = (h->speculative && !h->factored_exact) ? h->halo : 0;
  h->tri.launches = 0;
  h->tri.factor(H, s);
  h->factor_launches = h->tri.launches;
}

}  // namespace

extern "C" {

const char* psg_version(void) { return "psg-b200 0.1 (sm_100a)"; }

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
    std::copy(P.body_begin.begin(), P.body_begin.end(), body_begin);
    std::copy(P.body_end.begin(), P.body_end.end(), body_end);
    std::copy(P.sep_start.begin(), P.sep_start.end(), sep_start);
    *sep_count = (int)P.sep_start.size();
    *sep_size = P.sep_size;
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_factor(const psg_desc* Ain, int p, int strategy, double tol, void* stream, psg_handle** out, char* err,
               size_t errlen) {
  (void)tol;
  *out = nullptr;
  std::unique_ptr<psg_handle> h(new psg_handle);
  try {
    validate(*Ain);
    check_strategy(*Ain, strategy);
    h->plan = make_plan(*Ain, p);
    if (!is_tridiag(*Ain))
      throw Fail{PSG_E_UNSUPPORTED_KIND, "GPU path for this kind is not built yet (tridiagonal only)"};
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, s));
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
    refine_segments(h->plan, h->seg_start, h->seg_len, h->refined);
    h->tri.build(tri_rows(h->A), h->A.n, h->seg_start, h->seg_len);
    h->d_status.alloc(1);
    CUDA_TRY(cudaMallocHost(&h->h_status, sizeof(DevStatus)));
    run_factor(h.get(), s);
    CUDA_TRY(cudaEventRecord(e1, s));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    h->factor_seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out = h.release();
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

void psg_release(psg_handle* h) { delete h; }

int psg_set_option(psg_handle* h, int option, double value) {
  std::lock_guard<std::mutex> g(h->mu);
  switch (option) {
    case PSG_OPT_SPECULATIVE: h->speculative = value != 0.0; break;
    case PSG_OPT_HALO: h->halo = std::max(1, (int)value); break;
    case PSG_OPT_CERT_TOL: h->cert_tol = value; break;
    default: return 1 + PSG_E_INVALID_PARAMETER;
  }
  return 0;
}

int psg_last_launches(const psg_handle* h, int* f, int* s) {
  if (f) *f = h->factor_launches;
  if (s) *s = h->solve_launches;
  return 0;
}

int psg_solve(const psg_handle* hc, const double* f, double* x, int on_device, void* stream, psg_stats* stats,
              char* err, size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    const int n = h->A.n;
    const double* df = f;
    double* dx = x;
    if (!on_device) {
      h->d_f.alloc(n);
      h->d_x.alloc(n);
      CUDA_TRY(cudaMemcpyAsync(h->d_f.p, f, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      df = h->d_f.p;
      dx = h->d_x.p;
    }
    cudaEvent_t ev[4];
    const bool timing = stats != nullptr;
    if (timing)
      for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
    int fallbacks = 0;
    bool spec_used = false;
    double cert = 0;
    h->tri.launches = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      const bool spec = h->speculative && !h->factored_exact;
      const int H = spec ? h->halo : 0;
      DevStatus init{0ull, INT_MAX, 0};
      *h->h_status = init;
      CUDA_TRY(cudaMemcpyAsync(h->d_status.p, h->h_status, sizeof(DevStatus), cudaMemcpyHostToDevice, s));
      if (timing) CUDA_TRY(cudaEventRecord(ev[0], s));
      h->tri.solve(RowArr{df, 0, n}, dx, H, h->d_status.p, s, timing ? ev : nullptr);
      if (timing) CUDA_TRY(cudaEventRecord(ev[3], s));
      CUDA_TRY(cudaMemcpyAsync(h->h_status, h->d_status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      const DevStatus st = *h->h_status;
      cert = bits_to_double(st.cert_bits);
      const bool bad = st.bad_seg != INT_MAX;
      if (!bad && cert <= h->cert_tol) {
        spec_used = spec;
        break;
      }
      if (!spec) {
        if (bad) {
          // map the segment back to its reference partition (1-based)
          const int seg_row = h->seg_start[std::min<size_t>(st.bad_seg, h->seg_start.size() - 1)];
          int part = 1;
          for (int i = 0; i < h->plan.p; ++i)
            if (h->plan.body_begin[i] <= seg_row) part = i + 1;
          throw Fail{PSG_E_ZERO_PIVOT, "partition " + std::to_string(part) +
                                           ": zero pivot (non-finite value in the no-pivot elimination)"};
        }
        break;  // exact mode: report the certificate, keep the result
      }
      // speculative interface rejected: refactor exactly and re-solve
      ++fallbacks;
      h->factored_exact = true;
      run_factor(h, s);
    }
    if (!on_device) {
      CUDA_TRY(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    h->solve_launches = h->tri.launches;
    if (timing) {
      float t01 = 0, t12 = 0, t23 = 0;
      cudaEventElapsedTime(&t01, ev[0], ev[1]);
      cudaEventElapsedTime(&t12, ev[1], ev[2]);
      cudaEventElapsedTime(&t23, ev[2], ev[3]);
      stats->factor_seconds = h->factor_seconds;
      stats->phase1_seconds = t01 * 1e-3;
      stats->phase2_seconds = t12 * 1e-3;
      stats->phase3_seconds = t23 * 1e-3;
      stats->reduced_ops = h->tri.reduced_ops();
      stats->certificate = cert;
      stats->speculative = spec_used ? 1 : 0;
      stats->fallbacks = fallbacks;
      for (auto& e : ev) cudaEventDestroy(e);
    }
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_reduced_info(const psg_handle* h, int* q, int* dim, int* k, int* has_corner) {
  const int qq = (int)h->plan.sep_start.size();
  if (q) *q = qq;
  if (dim) *dim = qq * h->plan.sep_size;
  if (k) *k = h->plan.sep_size;
  if (has_corner) *has_corner = h->plan.has_corner ? 1 : 0;
  return 0;
}

int psg_reduced_blocks(const psg_handle* hc, double* diag, double* sub, double* super, char* err, size_t errlen) {
  psg_handle* h = const_cast<psg_handle*>(hc);
  std::lock_guard<std::mutex> g(h->mu);
  try {
    if (h->refined) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "reduced system was refined internally (bodies > 1088 rows)"};
    TriLevel& L = *h->tri.lv[0];
    const int ns = L.nseg - 1;
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
  std::lock_guard<std::mutex> g(h->mu);
  try {
    if (h->refined) throw Fail{PSG_E_UNSUPPORTED_STRUCTURE, "reduced system was refined internally (bodies > 1088 rows)"};
    cudaStream_t s = (cudaStream_t)stream;
    const int q = h->tri.lv[0]->nseg - 1;
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
    if (h->tri.lv.size() < 2) throw Fail{PSG_E_INVALID_PARAMETER, "no reduced system"};
    // The reduced system is level 1 of the solver; solve it in exact mode.
    h->tri.solve(RowArr{r, 0, q}, xo, 0, nullptr, s, nullptr, 1);
    // level 1's x output is xo; restore the level-0 wiring for later solves
    h->tri.lv[1]->x = h->tri.lv[0]->x_next.p;
    h->tri.lv[1]->F = RowArr{h->tri.lv[0]->rhs_next.p, 0, q};
    if (!on_device) CUDA_TRY(cudaMemcpyAsync(x, xo, sizeof(double) * q, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (stats) stats->reduced_ops += h->tri.reduced_ops();
    return 0;
  } catch (const Fail& f_) {
    return set_err(err, errlen, f_.code, f_.msg);
  }
}

int psg_matvec(const psg_desc* A, const double* x, double* y, int on_device, void* stream, char* err, size_t errlen) {
  try {
    validate(*A);
    if (!on_device || !A->on_device) throw Fail{PSG_E_INVALID_PARAMETER, "psg_matvec needs device pointers"};
    MatView v{A->kind, A->n, A->m, A->s, A->r, A->data, A->corner, A->corner_rows, A->corner_cols};
    matvec_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(v, x, y);
    LAUNCH_CHECK();
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
