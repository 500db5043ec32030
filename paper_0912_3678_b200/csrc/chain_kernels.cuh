// chain_kernels.cuh -- the partition method for the BVP layout of BABD
// (Kind::Babd with s = m, r = 0; BASELINE config 4):
//
//   block row 0       [ Ba                 ...   Bb(corner) ]   BC row
//   block row b >= 1  [ ... S_b  R_b ... ]                        x_b = R_b^-1 (f_b - S_b x_{b-1})
//
// i.e. a block lower-bidiagonal chain closed by the boundary condition.
// Chunk boundaries sigma_j = 16 j (internal, independent of the reference
// plan) cut the chain into chunks; chunk j maps x_{sigma_j} to
//     x_{sigma_{j+1}} = Phi_j x_{sigma_j} + phi_j,
//     Phi_j = prod T_b, T_b = -R_b^-1 S_b    (the body's F T G coupling block,
//                                             src/localfact.cpp:182-225)
//     phi_j = the chain from 0 with f         (condense, src/localfact.cpp:765-781)
//
//   factor  chain_tm_kernel (ONE launch): per block T_b and M_b = R_b^-1 (one
//           block per lane, LU in registers), stored beside the data; Phi_j
//           by a shared-memory tree product.  The reduced system in x_sigma is
//           again a BVP-layout chain (maps Phi_j, R = I, same Ba / Bb); its
//           chunk products Phi^(l) on every level are formed inside the same
//           launch by the warp that completes each chunk, and the last one
//           factors the top-level BC matrix (partial pivoting).
//   solve   chain_solve_kernel<0/1/2> (three launches): condense + reduced
//           levels up; top solve + x down + separator residuals up; the
//           correction down + certificate (see the kernel comment below).
//
#pragma once

#include "psg_common.cuh"

namespace psg {

// level 0: data = [Ba (MB*MB) | rows b = 1..nb-1: S_b | R_b (MB x 2MB, row-major)]
struct ChainLevelArgs {
  const double* data;
  const double* corner;  // Bb (MB x MB)
  int nb;                // block rows
  const double* f;       // rhs (nb * MB)
  double* x;             // solution
  double* tm;            // factor output / solve input: per block [T | M] (T = -R^-1 S, M = R^-1), row pairs interleaved (see the factor)
  DevStatus* status;
};

template <int MB>
__device__ __forceinline__ double gshfl(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src, MB);
}

template <int MB>
__device__ __forceinline__ void load_row(const double* data, int b, int i, double (&S)[MB], double (&R)[MB]) {
  const double* p = data + MB * MB + (long)(b - 1) * 2 * MB * MB + (long)i * 2 * MB;
#pragma unroll
  for (int c = 0; c < MB; ++c) {
    S[c] = __ldg(p + c);
    R[c] = __ldg(p + MB + c);
  }
}

__device__ __forceinline__ void cert_push(DevStatus* st, double num, double den) {
  double om = den > 0 ? num / den : num;
  if (!(om <= 1.0e308)) om = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) om = fmax(om, __shfl_xor_sync(0xffffffffu, om, o));
  if ((threadIdx.x & 31) == 0 && om > 0) status_cert(st, om);
}

// ---------------------------------------------------------------------------
// factor: per block b the transfer T_b = -R_b^-1 S_b and M_b = R_b^-1, stored
// row-interleaved like the data ([T row i | M row i], 2 MB doubles per row),
// and per chunk Phi_j = T_last ... T_first by a shared-memory tree product.
// One lane per block (LU in registers, no communication); a warp owns 32
// consecutive blocks = kChainC0-block chunks, staged through shared memory with
// a padded slot pitch (2 MB^2 + 2 doubles: conflict-free LDS.128 phases).
// ---------------------------------------------------------------------------
constexpr int kChainC0 = 16;  // chunk length (blocks) on every level

template <int MB>
struct ChainSmem {
  static constexpr int SLOT = 2 * MB * MB + 2;
  static constexpr int WARP = 32 * SLOT;  // doubles per warp
};

// [T | M] of a block in the pair-interleaved order of the global tm array
// (and of a slot once its block is factored): element (i, c) at
// (c / 2) * 2 MB + 2 i + c % 2 -- double2 (i, c/2) transposed
template <int MB>
__host__ __device__ constexpr int tix(int i, int c) {
  return (c >> 1) * 2 * MB + 2 * i + (c & 1);
}

// ---------------------------------------------------------------------------
// The reduced-system hierarchy.  Level 0 is the user's chain (N + 1 block
// rows, P[0] = ceil(N / 16) chunks).  Level l >= 1 has nb_l = P[l-1] + 1
// unknowns (x at the level-(l-1) chunk boundaries), block maps Phi^(l-1)
// (R = I) and rhs F_l: F_l[0] = the BC rhs, F_l[j+1] = phi^(l-1)_j.  Level T,
// the first with nb_T - 1 <= 16, is solved directly: the BC matrix
// G = Ba + Bb Phi_total is factored (partial pivoting) by the factor kernel.
// Every level is built by ONE launch: the warp / CTA that completes the last
// input of a level-l chunk (arrival counters, self-resetting) goes on to
// condense that chunk, so the upward sweep needs no further launches; the
// downward sweep is done redundantly by every CTA of the next kernel along
// its own path from the top (<= 16 steps per level).
// ---------------------------------------------------------------------------
constexpr int kChainMaxLev = 8;

struct ChainTree {
  int T;                          // top level (>= 1)
  int P[kChainMaxLev];            // chunks of level l (maps Phi^(l)), l < T; P[T-1] = nb_T - 1 <= 16
  double* phi[kChainMaxLev];      // Phi^(l): P[l] x MB x MB row-major
  double* fl[kChainMaxLev + 1];   // F_l, l = 1..T (nb_l x MB)
  double* cfl[kChainMaxLev + 1];  // correction rhs, l = 1..T
  int* cnt;                       // arrival counters
  int coff[kChainMaxLev + 1];     // level-l counters at cnt + coff[l] (l = 1..T-1), the top one at coff[T]
  double* glu;                    // LU of G (MB x MB) followed by the MB pivot rows (as doubles)
  double* x1;                     // final: x at the level-1 unknowns (level-0 separators)
  double* xlev[2];                // down sweep (x, d): values at level min(2, T)
  double* xtop[2];                // down sweep (x, d): values at the top unknowns
};

// warp-level arrival: true for the warp that completes the count (it then
// sees every other arriver's writes)
__device__ __forceinline__ bool warp_last_arrive(int* ctr, int expected, int lane) {
  __threadfence();
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    last = atomicAdd(ctr, 1) == expected - 1;
    if (last) atomicExch(ctr, 0);  // reset for the next launch
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last) __threadfence();
  return last != 0;
}

// tree of products P = later * earlier over the kChainC0 slots of each of
// `nch` chunks (T parts of the padded slots); the product lands in the
// chunk's LAST slot.  One lane per (product, row): the result row overwrites
// that row of the later factor, which only this lane reads; the earlier
// factor is a previous round's result (read-only in this round).
template <int MB>
__device__ __forceinline__ void chain_tree16(double* sm, int nch, int lane) {
  constexpr int SLOT = ChainSmem<MB>::SLOT;
#pragma unroll 1
  for (int h = 1; h < kChainC0; h <<= 1) {
    const int pairs = kChainC0 / (2 * h);  // per chunk
    const int tasks = nch * pairs * MB;
    for (int task = lane; task < tasks; task += 32) {
      const int i = task % MB, pk = task / MB, c = pk / pairs, k = pk % pairs;
      const double* E = sm + (c * kChainC0 + 2 * k * h + h - 1) * SLOT;
      double* L = sm + (c * kChainC0 + 2 * k * h + 2 * h - 1) * SLOT;
      double a[MB], o[MB];
#pragma unroll
      for (int l = 0; l < MB; ++l) a[l] = L[tix<MB>(i, l)];
#pragma unroll
      for (int cc = 0; cc < MB; ++cc) {
        double acc = a[0] * E[tix<MB>(0, cc)];
#pragma unroll
        for (int l = 1; l < MB; ++l) acc = fma(a[l], E[tix<MB>(l, cc)], acc);
        o[cc] = acc;
      }
#pragma unroll
      for (int cc = 0; cc < MB; ++cc) L[tix<MB>(i, cc)] = o[cc];
    }
    __syncwarp();
  }
}

// maps src[s] (s < len, written by another warp of this launch) into the T
// parts of slots 0..15, identity beyond
template <int MB>
__device__ __forceinline__ void chain_load_maps(double* sm, const double* src, int len, int lane) {
  constexpr int SLOT = ChainSmem<MB>::SLOT, MM = MB * MB;
  for (int e = lane; e < kChainC0 * MM; e += 32) {
    const int s = e / MM, r = e % MM, i = r / MB, k = r % MB;
    sm[s * SLOT + tix<MB>(i, k)] = s < len ? __ldcg(src + (long)s * MM + r) : (i == k ? 1.0 : 0.0);
  }
  __syncwarp();
}

// top level: Phi_total = product of the top maps, G = Ba + Bb Phi_total, LU
// of G with partial pivoting (LAPACK convention: full-row swaps, pivot rows
// recorded), the multipliers below the diagonal
template <int MB>
__device__ void chain_top_factor(const ChainLevelArgs& g, const ChainTree& t, double* sm, int lane) {
  constexpr int SLOT = ChainSmem<MB>::SLOT, MM = MB * MB, GP = MB + 1;
  chain_load_maps<MB>(sm, t.phi[t.T - 1], t.P[t.T - 1], lane);
  chain_tree16<MB>(sm, 1, lane);
  double* G = sm + SLOT;
  if (lane < MB) {
    const int i = lane;
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      double v = __ldg(g.data + i * MB + c);
#pragma unroll
      for (int l = 0; l < MB; ++l) v = fma(__ldg(g.corner + i * MB + l), sm[(kChainC0 - 1) * SLOT + tix<MB>(l, c)], v);
      G[i * GP + c] = v;
    }
  }
  __syncwarp();
  if (lane == 0) {
    for (int k = 0; k < MB; ++k) {
      int p = k;
      for (int r = k + 1; r < MB; ++r)
        if (fabs(G[r * GP + k]) > fabs(G[p * GP + k])) p = r;
      if (p != k)
        for (int c = 0; c < MB; ++c) {
          const double tmp = G[k * GP + c];
          G[k * GP + c] = G[p * GP + c];
          G[p * GP + c] = tmp;
        }
      t.glu[MM + k] = (double)p;
      for (int r = k + 1; r < MB; ++r) {
        const double l = G[r * GP + k] / G[k * GP + k];
        G[r * GP + k] = l;
        for (int c = k + 1; c < MB; ++c) G[r * GP + c] = fma(-l, G[k * GP + c], G[r * GP + c]);
      }
    }
    for (int e = 0; e < MM; ++e) t.glu[e] = G[(e / MB) * GP + e % MB];
  }
}

// after the level-0 chunk maps of warp w are stored: climb the hierarchy while
// this warp is the last arriver of the enclosing chunk
template <int MB>
__device__ void chain_factor_up(const ChainLevelArgs& g, const ChainTree& t, double* sm, long w, int lane) {
  constexpr int SLOT = ChainSmem<MB>::SLOT, MM = MB * MB;
  const long nw = ((long)t.P[0] + 1) / 2;  // factor warps (2 level-0 chunks each)
  long c = w;
  for (int l = 1;; ++l) {
    if (l == t.T) {
      const int expected = t.T == 1 ? (int)nw : t.P[t.T - 1];
      if (warp_last_arrive(t.cnt + t.coff[t.T], expected, lane)) chain_top_factor<MB>(g, t, sm, lane);
      return;
    }
    const long cc = l == 1 ? c / 8 : c / kChainC0;
    const int expected = l == 1 ? (int)min(8L, nw - 8 * cc) : (int)min((long)kChainC0, t.P[l - 1] - kChainC0 * cc);
    if (!warp_last_arrive(t.cnt + t.coff[l] + cc, expected, lane)) return;
    const int len = (int)min((long)kChainC0, t.P[l - 1] - kChainC0 * cc);
    chain_load_maps<MB>(sm, t.phi[l - 1] + kChainC0 * cc * MM, len, lane);
    chain_tree16<MB>(sm, 1, lane);
    for (int e = lane; e < MM; e += 32) t.phi[l][cc * MM + e] = sm[(kChainC0 - 1) * SLOT + tix<MB>(e / MB, e % MB)];
    c = cc;
  }
}

template <int MB>
__global__ void __launch_bounds__(64) chain_tm_kernel(ChainLevelArgs g, ChainTree t) {
  constexpr int SLOT = ChainSmem<MB>::SLOT, RW = 2 * MB, BW = 2 * MB * MB;
  extern __shared__ __align__(16) double csm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* sm = csm + wib * ChainSmem<MB>::WARP;
  const long w = (long)blockIdx.x * (blockDim.x >> 5) + wib;
  const long bfirst = 32 * w + 1;  // blocks bfirst .. bfirst + 31 (chunks 2w, 2w + 1)
  if (bfirst > g.nb - 1) return;   // warp-uniform
  const int nblk = (int)min(32L, g.nb - bfirst);
  // ---- stage the warp's blocks into padded slots: one TMA bulk copy per lane
  __shared__ __align__(8) uint64_t tbar[2];
  uint64_t* bar = tbar + wib;
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_arrive_expect_tx(bar, (uint32_t)nblk * BW * 8);
  }
  __syncwarp();
  if (lane < nblk) bulk_g2s(sm + lane * SLOT, g.data + MB * MB + (bfirst - 1 + lane) * BW, BW * 8, bar);
  mbar_wait(bar, 0);
  // ---- per lane: M = R^-1 (Gauss-Jordan, no pivoting), then T = -M S
  double* slot = sm + lane * SLOT;
  if (lane < nblk) {
    double R[MB * MB];
#pragma unroll
    for (int i = 0; i < MB; ++i)
#pragma unroll
      for (int c = 0; c < MB; ++c) R[(i) * MB + (c)] = slot[i * RW + MB + c];
    // M = R^-1 by in-place Gauss-Jordan (no pivoting, like the reference's Lu):
    // MB dependent pivot steps of MB^2 independent updates; stored over R
#pragma unroll
    for (int k = 0; k < MB; ++k) {
      const double p = fast_rcp(R[k * MB + k]);
      double col[MB], row[MB];
#pragma unroll
      for (int i = 0; i < MB; ++i) col[i] = R[i * MB + k];
#pragma unroll
      for (int j = 0; j < MB; ++j) row[j] = R[k * MB + j] * p;
#pragma unroll
      for (int i = 0; i < MB; ++i)
#pragma unroll
        for (int j = 0; j < MB; ++j) {
          if (i == k)
            R[i * MB + j] = j == k ? p : row[j];
          else
            R[i * MB + j] = j == k ? -col[i] * p : fma(-col[i], row[j], R[i * MB + j]);
        }
    }
    double (&Mi)[MB * MB] = R;
#pragma unroll
    for (int i = 0; i < MB; ++i)
#pragma unroll
      for (int c = 0; c < MB; ++c) slot[i * RW + MB + c] = Mi[i * MB + c];
    // T = -M S column by column (independent FMA chains), stored over S
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      double sc[MB];
#pragma unroll
      for (int l = 0; l < MB; ++l) sc[l] = slot[l * RW + c];
#pragma unroll
      for (int i = 0; i < MB; ++i) {
        double acc = -Mi[i * MB] * sc[0];
#pragma unroll
        for (int l = 1; l < MB; ++l) acc = fma(-Mi[i * MB + l], sc[l], acc);
        slot[i * RW + c] = acc;
      }
    }
    // ---- pair-interleave the slot in place (double2 (i, q) <-> (q, i)), then
    // one TMA bulk store of the block: block b, double2 q*MB + i = row i,
    // columns 2q, 2q+1 of [T | M] -- the solve's MB lanes read one contiguous
    // MB*16-byte run per load (coalesced)
    double2* s2 = reinterpret_cast<double2*>(slot);
#pragma unroll
    for (int i = 0; i < MB; ++i)
#pragma unroll
      for (int q = i + 1; q < MB; ++q) {
        const double2 x = s2[i * MB + q], y = s2[q * MB + i];
        s2[i * MB + q] = y;
        s2[q * MB + i] = x;
      }
    fence_proxy_async_smem();
    bulk_s2g(g.tm + (bfirst - 1 + lane) * BW, slot, BW * 8);
    bulk_commit_and_wait_read();
  } else {  // missing blocks of a short last chunk: T = I
#pragma unroll
    for (int i = 0; i < MB; ++i)
#pragma unroll
      for (int c = 0; c < MB; ++c) slot[tix<MB>(i, c)] = i == c ? 1.0 : 0.0;
  }
  __syncwarp();
  // ---- Phi of the two chunks: tree of products P = later * earlier, in the T slots
  chain_tree16<MB>(sm, 2, lane);
  // ---- Phi^(0) of this warp's chunks, then the upper levels of the hierarchy
  const long P0 = t.P[0];
  for (int e = lane; e < 2 * MB * MB; e += 32) {
    const int c = e / (MB * MB), r = e % (MB * MB);
    if (2 * w + c < P0)
      t.phi[0][(2 * w + c) * MB * MB + r] = sm[(c * kChainC0 + kChainC0 - 1) * SLOT + tix<MB>(r / MB, r % MB)];
  }
  chain_factor_up<MB>(g, t, sm, w, lane);
}

// ---------------------------------------------------------------------------
// solve: three launches of chain_solve_kernel<MB, KM>, one CTA per level-1
// chunk c (16 level-0 chunks, MB lanes each: lane i = row i of every block).
//   KM 0 (condense)   level-0 chunks: phi_j = chain from zero with f; the CTA
//                     condenses its level-1 chunk, last arrivers the upper ones.
//   KM 1 (final)      warp 0 solves the top level and walks down its own path
//                     (<= 16 steps per level) to x at its 17 level-1 unknowns;
//                     level-0 chunks: x through every block from x_sigma, the
//                     separator rows' residuals condensed to R^-1 r (the chain's
//                     end value differs from the affine map by rounding, ~8 eps
//                     |x| per step) and the BC row residual; these rhs go up
//                     the hierarchy like KM 0.
//   KM 2 (correction) the correction d the same way down; x += the homogeneous
//                     chain of d, certificate of the corrected separator rows
//                     and of the BC row.
// Level-0 passes read row i of [T | M] (pair-interleaved: each load of a
// group is one contiguous run) and f, kPre steps ahead in a register ring inside a fully
// unrolled kChainC0-step chain.
// ---------------------------------------------------------------------------
constexpr int kPre = 3;

template <int MB>
struct ChainReg {  // staged maps (padded rows: conflict-free) + rhs slots of one <= 16-step chain
  static constexpr int MP = MB + 1;
  static constexpr int MAPS = kChainC0 * MB * MP;
  static constexpr int SIZE = MAPS + (kChainC0 + 1) * MB;
};

// maps[first + s] (s < len) and rhs[rfirst + s] (s < nr); cooperative over nthr threads
template <int MB, bool COHERENT_RHS>
__device__ __forceinline__ void chain_stage(double* reg, const double* maps, long first, int len, const double* rhs,
                                            long rfirst, int nr, int tid, int nthr) {
  constexpr int MM = MB * MB, MP = MB + 1;
  for (int e = tid; e < len * MM; e += nthr) {
    const int s = e / MM, r = e % MM;
    reg[s * MB * MP + (r / MB) * MP + r % MB] = __ldg(maps + (first + s) * MM + r);
  }
  double* rr = reg + ChainReg<MB>::MAPS;
  for (int e = tid; e < nr * MB; e += nthr)
    rr[e] = COHERENT_RHS ? __ldcg(rhs + rfirst * MB + e) : __ldg(rhs + rfirst * MB + e);
}

// y <- map_s y + fi (row i)
template <int MB>
__device__ __forceinline__ double chain_step(const double* reg, int s, int i, double y, double fi) {
  const double* m = reg + s * MB * (MB + 1) + i * (MB + 1);
  double a0 = fi, a1 = 0.0;
#pragma unroll
  for (int l = 0; l < MB; l += 2) {
    a0 = fma(m[l], gshfl<MB>(y, l), a0);
    a1 = fma(m[l + 1], gshfl<MB>(y, l + 1), a1);
  }
  return a0 + a1;
}

// condense a staged chunk of len steps from zero
template <int MB>
__device__ __forceinline__ double chain_condense(const double* reg, int len, int i) {
  const double* rr = reg + ChainReg<MB>::MAPS;
  double y = 0.0;
  for (int s = 1; s <= len; ++s) y = chain_step<MB>(reg, s - 1, i, y, rr[s * MB + i]);
  return y;
}

// level-0 chunk j: MODE 0 condense (run returns phi_j), 1 final, 2 correction.
// start() issues the first kPre steps' loads (callers do it before their
// serial prologue so the loads are in flight meanwhile).
template <int MB, int MODE>
struct Pass0 {
  long b0 = 0;
  int len = 0;
  double Tq[kPre][MB], Mq[kPre][MB], Fq[kPre], Xq[kPre];  // Fq: f_i of the block (row i; shuffled for M f)

  __device__ __forceinline__ void fetch(const ChainLevelArgs& g, int i, int t, int slot) {
    constexpr int BW = 2 * MB * MB;
    if (t < len) {
      const double2* row = reinterpret_cast<const double2*>(g.tm + (b0 + t - 1) * BW) + i;
#pragma unroll
      for (int c = 0; c < MB / 2; ++c) {
        const double2 tv = __ldg(row + c * MB);
        Tq[slot][2 * c] = tv.x;
        Tq[slot][2 * c + 1] = tv.y;
      }
      if (MODE != 2) {
#pragma unroll
        for (int c = 0; c < MB / 2; ++c) {
          const double2 mv = __ldg(row + (MB / 2 + c) * MB);
          Mq[slot][2 * c] = mv.x;
          Mq[slot][2 * c + 1] = mv.y;
        }
        Fq[slot] = __ldg(g.f + (b0 + t) * MB + i);
      } else {
        Xq[slot] = g.x[(b0 + t) * MB + i];
      }
    }
  }

  __device__ __forceinline__ void start(const ChainLevelArgs& g, long j, bool live, int i) {
    b0 = kChainC0 * j + 1;
    const long b1 = live ? min(kChainC0 * j + kChainC0, (long)g.nb - 1) : 0;
    len = live ? (int)(b1 - b0 + 1) : 0;
#pragma unroll
    for (int t = 0; t < kPre; ++t) fetch(g, i, t, t);
  }

  __device__ __forceinline__ double run(const ChainLevelArgs& g, long j, bool live, int i, double ys, double yts,
                                        double ye, double yte, double& corr, double& num, double& den,
                                        bool& finite) {
    double y = ys, yt = yts;
    if (MODE != 0 && live && j == 0) g.x[i] = yt;
#pragma unroll
    for (int t = 0; t < kChainC0; ++t) {
      const int sl = t % kPre;
      const bool act = t < len, last = t == len - 1;
      double a = 0.0;
      if (MODE != 2)
#pragma unroll
        for (int l = 0; l < MB; ++l) a = fma(Mq[sl][l], gshfl<MB>(Fq[sl], l), a);
#pragma unroll
      for (int l = 0; l < MB; ++l) a = fma(Tq[sl][l], gshfl<MB>(y, l), a);
      const double xold = MODE == 2 ? Xq[sl] : 0.0;
      // correction: certificate of the corrected separator row r = f - S x_prev - R x_sep
      double S[MB], R[MB];
      const bool cert_here = MODE == 2 && act && last;
      if (cert_here) load_row<MB>(g.data, b0 + t, i, S, R);
      double sg = 0.0, ab = 0.0;
      if (MODE == 2) {
#pragma unroll
        for (int l = 0; l < MB; ++l) {
          const double pl = gshfl<MB>(yt, l);
          if (cert_here) {
            const double p1 = S[l] * pl;
            sg += p1;
            ab += fabs(p1);
          }
        }
      }
      if (act) {
        const long os = (b0 + t) * MB + i;
        if (!last) {
          y = a;
          yt = MODE == 2 ? xold + y : y;
        } else if (MODE == 1) {
          corr = a - ye;  // R^-1 r_sep
          y = yt = ye;
        } else if (MODE == 2) {
          y = ye;
          yt = yte;
        } else {
          y = a;
        }
        if (MODE != 0) {
          g.x[os] = yt;
          finite &= isfinite(yt);
        }
      }
      if (t + kPre < kChainC0) fetch(g, i, t + kPre, sl);
      if (MODE == 2) {
#pragma unroll
        for (int l = 0; l < MB; ++l) {
          const double xl = gshfl<MB>(yt, l);
          if (cert_here) {
            const double p2 = R[l] * xl;
            sg += p2;
            ab += fabs(p2);
          }
        }
        if (cert_here) {
          const double fv = __ldg(g.f + (b0 + t) * MB + i);
          const double on = fabs(fv - sg), od = fabs(fv) + ab;
          if (on * den > num * od || (den == 0.0 && on > 0)) {
            num = on;
            den = od;
          }
        }
      }
    }
    return y;
  }
};

// upward sweep from the CTA's level-1 chunk (reg1: its maps, rhs slots = F_1
// of the chunk): F_2[c+1], then every level whose chunk this warp completes
template <int MB>
__device__ void chain_up(const ChainTree& t, double* const* Fu, double* reg1, long c, int len1, int lane) {
  const int i = lane % MB;
  const double* rr = reg1 + ChainReg<MB>::MAPS;
  double y = chain_condense<MB>(reg1, len1, i);
  if (lane < MB) {
    Fu[2][(c + 1) * MB + i] = y;
    if (c == 0) Fu[2][i] = rr[i];
  }
  long prev = c;
  for (int l = 2; l < t.T; ++l) {
    const long cc = prev / kChainC0;
    const int len = (int)min((long)kChainC0, t.P[l - 1] - kChainC0 * cc);
    if (!warp_last_arrive(t.cnt + t.coff[l] + cc, len, lane)) return;
    chain_stage<MB, true>(reg1, t.phi[l - 1], kChainC0 * cc, len, Fu[l], kChainC0 * cc, len + 1, lane, 32);
    __syncwarp();
    y = chain_condense<MB>(reg1, len, i);
    if (lane < MB) {
      Fu[l + 1][(cc + 1) * MB + i] = y;
      if (cc == 0) Fu[l + 1][i] = rr[i];
    }
    __syncwarp();
    prev = cc;
  }
}

// top level of a sweep: phi_total, x_0 from G x_0 = F_T[0] - Bb phi_total
// (stored LU, pivots), the top chain; values into s_top (whole warp)
template <int MB>
__device__ void chain_top_solve(const ChainLevelArgs& g, const ChainTree& t, const double* regT, const double* s_glu,
                                double* s_r, double* s_top, int lane) {
  constexpr int MM = MB * MB;
  const int i = lane % MB, PT = t.P[t.T - 1];
  const double* rT = regT + ChainReg<MB>::MAPS;
  double y = chain_condense<MB>(regT, PT, i);
  double r = rT[i];
#pragma unroll
  for (int l = 0; l < MB; ++l) r = fma(-__ldg(g.corner + i * MB + l), gshfl<MB>(y, l), r);
  if (lane < MB) s_r[i] = r;
  __syncwarp();
  if (lane == 0) {
    for (int k = 0; k < MB; ++k) {
      const int p = (int)s_glu[MM + k];
      if (p != k) {
        const double tmp = s_r[k];
        s_r[k] = s_r[p];
        s_r[p] = tmp;
      }
    }
    for (int k = 0; k < MB; ++k)
      for (int rr = k + 1; rr < MB; ++rr) s_r[rr] = fma(-s_glu[rr * MB + k], s_r[k], s_r[rr]);
    for (int k = MB - 1; k >= 0; --k) {
      double sv = s_r[k];
      for (int cc = k + 1; cc < MB; ++cc) sv = fma(-s_glu[k * MB + cc], s_r[cc], sv);
      s_r[k] = sv / s_glu[k * MB + k];
    }
  }
  __syncwarp();
  y = s_r[i];
  if (lane < MB) s_top[i] = y;
  for (int s = 1; s <= PT; ++s) {
    y = chain_step<MB>(regT, s - 1, i, y, rT[s * MB + i]);
    if (lane < MB) s_top[s * MB + i] = y;
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// down sweep (one warp per level-2 chunk w; one warp when T <= 2): the top
// solve and this warp's path down to the values at its level-2 chunk
// (<= 16 steps per level), written to t.xlev[sel]; warp 0 also writes the top
// values.  sel 0: x (rhs F), 1: the correction d (rhs cF).
// ---------------------------------------------------------------------------
template <int MB>
__global__ void __launch_bounds__(32) chain_down_kernel(ChainLevelArgs g, ChainTree t, int sel) {
  constexpr int REG = ChainReg<MB>::SIZE, MAPS = ChainReg<MB>::MAPS, MM = MB * MB;
  extern __shared__ __align__(16) double ssm[];
  __shared__ double s_top[(kChainC0 + 1) * MB];
  __shared__ double s_glu[MM + MB];
  __shared__ double s_r[MB];
  const int lane = threadIdx.x, i = lane % MB, T = t.T, PT = t.P[T - 1];
  const long w = blockIdx.x;
  double* const* F = sel ? t.cfl : t.fl;
  // regions: top at ssm, level l (2 <= l < T) at ssm + (T - l) * REG
  chain_stage<MB, false>(ssm, t.phi[T - 1], 0, PT, F[T], 0, PT + 1, lane, 32);
  for (int l = 2; l < T; ++l) {
    const long cc = w >> (4 * (l - 2));
    const int len = (int)min((long)kChainC0, t.P[l - 1] - kChainC0 * cc);
    chain_stage<MB, false>(ssm + (T - l) * REG, t.phi[l - 1], kChainC0 * cc, len, F[l], kChainC0 * cc, len + 1, lane,
                           32);
  }
  for (int e = lane; e < MM + MB; e += 32) s_glu[e] = __ldg(t.glu + e);
  __syncwarp();
  chain_top_solve<MB>(g, t, ssm, s_glu, s_r, s_top, lane);
  double* out = t.xlev[sel];
  if (w == 0 && lane < MB)
    for (int s = 0; s <= PT; ++s) t.xtop[sel][s * MB + i] = s_top[s * MB + i];
  if (T <= 2) {  // the top level is level min(2, T) itself
    if (lane < MB)
      for (int s = 0; s <= PT; ++s) out[s * MB + i] = s_top[s * MB + i];
    return;
  }
  const long uT = w >> (4 * (T - 3));
  double lo = s_top[uT * MB + i], hi = s_top[(uT + 1) * MB + i];
  for (int l = T - 1; l >= 3; --l) {
    const long ul = w >> (4 * (l - 3)), cc = ul >> 4;
    const int t0 = (int)(ul & 15), len = (int)min((long)kChainC0, t.P[l - 1] - kChainC0 * cc);
    const double* R = ssm + (T - l) * REG;
    const double* Rr = R + MAPS;
    double yy = lo;
    for (int s = 1; s <= t0; ++s) yy = chain_step<MB>(R, s - 1, i, yy, Rr[s * MB + i]);
    hi = t0 + 1 == len ? hi : chain_step<MB>(R, t0, i, yy, Rr[(t0 + 1) * MB + i]);
    lo = yy;
  }
  // level-2 chunk w
  const double* R = ssm + (T - 2) * REG;
  const double* Rr = R + MAPS;
  const int len2 = (int)min((long)kChainC0, t.P[1] - kChainC0 * w);
  double yy = lo;
  if (lane < MB) out[kChainC0 * w * MB + i] = lo;
  for (int s = 1; s < len2; ++s) {
    yy = chain_step<MB>(R, s - 1, i, yy, Rr[s * MB + i]);
    if (lane < MB) out[(kChainC0 * w + s) * MB + i] = yy;
  }
  if (lane < MB && kChainC0 * w + len2 == t.P[1]) out[(long)t.P[1] * MB + i] = hi;
}

template <int MB, int KM>
__global__ void __launch_bounds__(16 * MB) chain_solve_kernel(ChainLevelArgs g, ChainTree t) {
  constexpr int NT = 16 * MB, MAPS = ChainReg<MB>::MAPS, MM = MB * MB;
  extern __shared__ __align__(16) double ssm[];
  __shared__ double s_v[(kChainC0 + 1) * MB];  // x (KM 1) or d (KM 2) at this CTA's level-1 unknowns
  __shared__ double s_x[(kChainC0 + 1) * MB];  // KM 2: x at the level-1 unknowns
  const int tid = threadIdx.x, lane = tid & 31, grp = tid / MB, i = tid % MB;
  const long c = blockIdx.x;
  const int T = t.T;
  const long P0 = t.P[0];
  const long j = kChainC0 * c + grp;
  const bool live = j < P0;
  const int len1 = (int)min((long)kChainC0, P0 - kChainC0 * c);
  double* reg1 = ssm;  // level-1 region: maps Phi^(0) of this CTA's chunk + rhs slots
  double* rr1 = reg1 + MAPS;
  double num = 0.0, den = 0.0, corr = 0.0;
  bool finite = true;
  (void)MM;

  if constexpr (KM == 0) {
    Pass0<MB, 0> ps;
    ps.start(g, j, live, i);
    if (T >= 2) chain_stage<MB, false>(reg1, t.phi[0], kChainC0 * c, len1, nullptr, 0, 0, tid, NT);
    const double y = ps.run(g, j, live, i, 0.0, 0.0, 0.0, 0.0, corr, num, den, finite);
    if (live) {
      t.fl[1][(j + 1) * MB + i] = y;
      rr1[(grp + 1) * MB + i] = y;
      if (j == 0) {
        const double f0 = __ldg(g.f + i);
        t.fl[1][i] = f0;
        rr1[i] = f0;
      }
    }
    if (T < 2) return;
    __syncthreads();
    if (tid < 32) chain_up<MB>(t, t.fl, reg1, c, len1, lane);
  } else {
    constexpr int SEL = KM == 1 ? 0 : 1;
    double* const* Fd = SEL ? t.cfl : t.fl;  // rhs of the level-1 chain
    Pass0<MB, KM> ps;
    ps.start(g, j, live, i);
    if (T >= 2) chain_stage<MB, false>(reg1, t.phi[0], kChainC0 * c, len1, Fd[1], kChainC0 * c, len1 + 1, tid, NT);
    if (KM == 2)
      for (int e = tid; e < (len1 + 1) * MB; e += NT) s_x[e] = __ldg(t.x1 + kChainC0 * c * MB + e);
    __syncthreads();
    if (tid < 32) {  // this CTA's level-1 values from the down sweep's level-2 values
      const double* xl = t.xlev[SEL];
      if (T == 1) {
        if (lane < MB)
          for (int s = 0; s <= len1; ++s) s_v[s * MB + i] = __ldg(xl + s * MB + i);
      } else {
        const double lo = __ldg(xl + c * MB + i), hi = __ldg(xl + (c + 1) * MB + i);
        double yy = lo;
        if (lane < MB) s_v[i] = lo;
        for (int s = 1; s < len1; ++s) {
          yy = chain_step<MB>(reg1, s - 1, i, yy, rr1[s * MB + i]);
          if (lane < MB) s_v[s * MB + i] = yy;
        }
        if (lane < MB) s_v[len1 * MB + i] = hi;
      }
    }
    __syncthreads();
    const int PT = t.P[T - 1];
    if constexpr (KM == 1) {
      ps.run(g, j, live, i, s_v[grp * MB + i], s_v[grp * MB + i], s_v[(grp + 1) * MB + i], s_v[(grp + 1) * MB + i],
             corr, num, den, finite);
      if (live) {
        t.x1[j * MB + i] = s_v[grp * MB + i];
        if (j + 1 == P0) t.x1[(j + 1) * MB + i] = s_v[(grp + 1) * MB + i];
        t.cfl[1][(j + 1) * MB + i] = corr;
        rr1[(grp + 1) * MB + i] = corr;
      }
      if (c == 0 && tid < 32) {  // BC row residual: F_0 - Ba x_0 - Bb x_N (every group runs the shuffles)
        const double x0 = s_v[i], xe = __ldg(t.xtop[0] + PT * MB + i);
        double sg = 0.0;
#pragma unroll
        for (int l = 0; l < MB; ++l) {
          const double a0 = gshfl<MB>(x0, l), ae = gshfl<MB>(xe, l);
          sg += __ldg(g.data + i * MB + l) * a0 + __ldg(g.corner + i * MB + l) * ae;
        }
        if (lane < MB) {
          const double r0 = __ldg(g.f + i) - sg;
          t.cfl[1][i] = r0;
          rr1[i] = r0;
        }
      }
      if (T < 2) return;
      __syncthreads();
      if (tid < 32) chain_up<MB>(t, t.cfl, reg1, c, len1, lane);
    } else {
      // x += the homogeneous chain of d; certificate
      const double d0 = s_v[grp * MB + i], d1 = s_v[(grp + 1) * MB + i];
      ps.run(g, j, live, i, d0, s_x[grp * MB + i] + d0, d1, s_x[(grp + 1) * MB + i] + d1, corr, num, den, finite);
      if (c == 0 && tid < 32) {  // BC row with the corrected end values
        const double x0 = __ldg(t.xtop[0] + i) + __ldg(t.xtop[1] + i);
        const double xe = __ldg(t.xtop[0] + PT * MB + i) + __ldg(t.xtop[1] + PT * MB + i);
        double sg = 0.0, ab = 0.0;
#pragma unroll
        for (int l = 0; l < MB; ++l) {
          const double p1 = __ldg(g.data + i * MB + l) * gshfl<MB>(x0, l);
          const double p2 = __ldg(g.corner + i * MB + l) * gshfl<MB>(xe, l);
          sg += p1 + p2;
          ab += fabs(p1) + fabs(p2);
        }
        const double fv = __ldg(g.f + i), on = fabs(fv - sg), od = fabs(fv) + ab;
        if (on * den > num * od || (den == 0.0 && on > 0)) {
          num = on;
          den = od;
        }
      }
      if (!finite) num = __longlong_as_double(0x7ff0000000000000ll), den = 1.0;
      if (g.status) cert_push(g.status, num, den);
    }
  }
}

}  // namespace psg
