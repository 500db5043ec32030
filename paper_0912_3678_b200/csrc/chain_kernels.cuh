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
//   factor + condense  chain_fc_kernel (ONE pass over A and f): per block
//           T_b = -R_b^-1 S_b and c_b = R_b^-1 f_b by Gauss-Jordan on the
//           augmented rows (MB lanes per block, row per lane), stored for the
//           final pass; the chunk maps (Phi_j, phi_j) composed on the fly.
//           The reduced system in x_sigma is again a BVP-layout chain (maps
//           Phi_j, R = I, same Ba / Bb); its chunk maps on every level are
//           composed inside the same launch by the CTA / composer that
//           completes each chunk, and the last one factors the top-level BC
//           matrix (partial pivoting).  The factor is lazy: a refactor
//           followed by a solve runs this one fused launch.
//   solve   chain_down_kernel (top solve + x down), chain_solve_kernel<1>
//           (x through every block, separator residuals up), chain_down_kernel
//           (the correction down), chain_solve_kernel<2> (x += d, certificate).
//
#pragma once

#include "psg_common.cuh"

namespace psg {

// -DPSG_PROF: %globaltimer stamps per kernel of a solve (tools/tl_probe.py):
// g_tl[id][k], id 0 factor, 1 / 3 down sweeps, 2 / 4 level-0 passes, 6 / 7
// inside the sweeps, 9.. the factor's upper levels, 12 its top LU.
#ifdef PSG_PROF
__device__ unsigned long long g_tl[16][4];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#define TL_MAX(id, k) \
  if (threadIdx.x == 0) atomicMax(&g_tl[id][k], tl_now())
#define TL_MIN(id, k) \
  if (threadIdx.x == 0) atomicMin(&g_tl[id][k], tl_now())
#else
#define TL_MAX(id, k)
#define TL_MIN(id, k)
#endif

// level 0: data = [Ba (MB*MB) | rows b = 1..nb-1: S_b | R_b (MB x 2MB, row-major)]
struct ChainLevelArgs {
  const double* data;
  const double* corner;  // Bb (MB x MB)
  int nb;                // block rows
  const double* f;       // rhs (nb * MB)
  double* x;             // solution
  double* tm;            // per block T_b = -R_b^-1 S_b (MB x MB, double2 (row i, columns 2q, 2q+1) at q MB + i)
  double* cv;            // condense output: per block c_b = R_b^-1 f_b (nb x MB, block 0 unused)
  DevStatus* status;
  DevStatus* host_out;  // pinned host slot the correction pass publishes the status to (NULL: none)
  unsigned* done_ctr;   // its arrival counter
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

constexpr int kChainC0 = 16;  // chunk length (blocks) on every level

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

// ---------------------------------------------------------------------------
// chain_fc_kernel: the level-0 factor and condense of the chain in ONE pass
// over A (and f), plus the whole reduced hierarchy.
//
// A subgroup of MB lanes owns one level-0 chunk (16 consecutive block rows),
// lane i = row i of every block.  Per block: [S | R] arrives by cp.async
// (16-byte pieces, coalesced, XOR-swizzled so each lane reads its row
// conflict-free), two blocks in flight per subgroup; Gauss-Jordan on the
// augmented rows [R | S | f] with the pivot row broadcast through shared
// memory leaves R diagonal, so T_b = -D^-1 S' and c_b = D^-1 f' (no pivoting,
// like the reference's Lu); lane i stores row i of T_b (pair-interleaved, the
// final pass reads it coalesced) and c_b.  The chunk's affine map
//     (Phi_j, phi_j) = (T_16, c_16) o ... o (T_1, c_1)
// accumulates as it goes: lane i keeps column i of Phi (Phi <- T_b Phi) and
// the whole phi (phi <- T_b phi + c_b), T_b read back from shared memory.
//
// A CTA (4 warps) holds 128 / MB chunks = 8 / MB level-1 chunks, which warp 0
// composes right away (maps from L2); higher levels and the top BC matrix
// G = Ba + Bb Phi_total (factored with partial pivoting) are done by the last
// arriving CTA / composer (self-resetting counters), all inside the launch.
//
// STORE_T: store T_b and the maps Phi (factor); WITH_F: c_b and phi (condense).
//   <true, true>   refactor + first solve fused (the production step)
//   <true, false>  factor alone
//   <false, true>  condense alone (a further right-hand side): A is read again
//                  instead of keeping R^-1 (same bytes as storing it)
// ---------------------------------------------------------------------------
template <int MB>
struct FcCfg {
  static constexpr int SG = 32 / MB;                                  // subgroups (chunks) per warp
  static constexpr int NW = 4;                                        // warps per CTA
  static constexpr int CPC = NW * SG;                                 // level-0 chunks per CTA
  static constexpr int L1C = CPC / kChainC0;                          // level-1 chunks per CTA (8 / MB)
  static constexpr int BLK = 2 * MB * MB;                             // [S | R] doubles per block row
  static constexpr int TP = MB + 2;                                   // row pitch of the published T_b
  static constexpr int PIV = 2 * MB + 2;                              // pivot row buffer
  static constexpr int TBS = MB * TP + MB;                            // published T_b + phi
  static constexpr int SUB = 2 * BLK + TBS + 2 * PIV;                 // doubles per subgroup
  static constexpr int SMEM = NW * SG * SUB * 8;                      // bytes per CTA
};

template <int MB>
__device__ __forceinline__ double pick(const double (&v)[MB], int i) {
  double o = 0.0;
#pragma unroll
  for (int r = 0; r < MB; ++r) o = r == i ? v[r] : o;
  return o;
}

// Combine the affine maps held by 16 consecutive subgroups of the CTA (map of
// subgroup s covers chunk range s; later o earlier) into the first subgroup of
// each group of 16: four rounds, the later partner publishes (Phi, phi) in its
// shared buffer, the earlier one composes Phi_L Phi_E (lane i: column i) and
// Phi_L phi_E + phi_L.  Every thread of the CTA calls it.
template <int MB, bool VEC>
__device__ __forceinline__ void fc_tree16(double* fsm, int gsub, int i, double (&pc)[MB], double (&ph)[MB]) {
  using C = FcCfg<MB>;
  const int s = gsub % kChainC0;
#pragma unroll 1
  for (int h = 1; h < kChainC0; h <<= 1) {
    double* mine = fsm + gsub * C::SUB + 2 * C::BLK;  // TB region: MB x TP, then MB for phi
    if (s % (2 * h) == h) {  // later partner of (s - h): publish
#pragma unroll
      for (int r = 0; r < MB; ++r) mine[r * C::TP + i] = pc[r];
      if (VEC) mine[MB * C::TP + i] = pick<MB>(ph, i);
    }
    __syncthreads();
    if (s % (2 * h) == 0) {
      const double* L = fsm + (gsub + h) * C::SUB + 2 * C::BLK;
      double np[MB], nv[MB];
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        double a = 0.0, v = VEC ? L[MB * C::TP + r] : 0.0;
#pragma unroll
        for (int c = 0; c < MB; c += 2) {
          const double2 m = *reinterpret_cast<const double2*>(L + r * C::TP + c);
          a = fma(m.y, pc[c + 1], fma(m.x, pc[c], a));
          if (VEC) v = fma(m.y, ph[c + 1], fma(m.x, ph[c], v));
        }
        np[r] = a;
        nv[r] = v;
      }
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        pc[r] = np[r];
        if (VEC) ph[r] = nv[r];
      }
    }
    __syncthreads();
  }
}

// top of the hierarchy: G = Ba + Bb Phi_total (lane i holds column i of
// Phi_total), LU with partial pivoting (full-row swaps, pivot rows recorded)
// into t.glu.  Lanes 0..MB-1 of one warp; G staged in `buf`.
template <int MB>
__device__ void chain_fc_top(const ChainLevelArgs& g, const ChainTree& t, double* buf, int lane, const double (&pc)[MB]) {
  constexpr int MM = MB * MB, GP = MB + 1;
  const int i = lane % MB;
  if (lane < MB) {
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      double v = __ldg(g.data + r * MB + i);
#pragma unroll
      for (int l = 0; l < MB; ++l) v = fma(__ldg(g.corner + r * MB + l), pc[l], v);
      buf[r * GP + i] = v;
    }
  }
  __syncwarp();
  if (lane == 0) {
    double* G = buf;
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
  __syncwarp();
}

// CTA-level arrival: true (for every thread) in the CTA that completes the count
__device__ __forceinline__ bool cta_last_arrive(int* ctr, int expected) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int last = atomicAdd(ctr, 1) == expected - 1;
    if (last) atomicExch(ctr, 0);  // reset for the next launch
    s_last = last;
  }
  __syncthreads();
  const bool last = s_last != 0;
  if (last) __threadfence();
  return last;
}

template <int MB, bool STORE_T, bool WITH_F>
__global__ void __launch_bounds__(128) chain_fc_kernel(ChainLevelArgs g, ChainTree t) {
  pdl_trigger();  // the down sweep may launch (it waits for this grid before reading anything)
  using C = FcCfg<MB>;
  constexpr int MM = MB * MB, RW = 2 * MB;
  extern __shared__ __align__(16) double fsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, sg = lane / MB, i = lane % MB;
  double* sub = fsm + (wid * C::SG + sg) * C::SUB;
  double* stage = sub;                       // 2 x BLK
  double* TB = sub + 2 * C::BLK;             // MB x TP published T_b, then phi
  double* PB = TB + C::TBS;                  // 2 pivot rows
  const long P0 = t.P[0];
  const long j = (long)blockIdx.x * C::CPC + wid * C::SG + sg;  // level-0 chunk
  const bool live = j < P0;
  const long nblk = (long)g.nb - 1;                             // blocks after the BC row
  const int len = live ? (int)min((long)kChainC0, nblk - kChainC0 * j) : 0;
  const long b0 = kChainC0 * j + 1;                             // first block row of the chunk
  auto issue = [&](int tt) {  // cp.async of block row b0 + tt into stage buffer tt & 1
    if (tt < len) {
      const double* src = g.data + MM + (b0 + tt - 1) * C::BLK;
      double* dst = stage + (tt & 1) * C::BLK;
#pragma unroll
      for (int q = 0; q < MB; ++q) cp_async16(dst + q * RW + 2 * (i ^ q), src + q * RW + 2 * i);
    }
    cp_async_commit();
  };
  double pc[MB], ph[MB];
#pragma unroll
  for (int r = 0; r < MB; ++r) {
    pc[r] = r == i ? 1.0 : 0.0;
    ph[r] = 0.0;
  }
  issue(0);
#pragma unroll 1
  for (int tt = 0; tt < kChainC0; ++tt) {
    issue(tt + 1);
    cp_async_wait<1>();
    __syncwarp();
    const bool act = tt < len;
    double R[MB], S[MB], fv = 0.0;
    {
      const double* row = stage + (tt & 1) * C::BLK + i * RW;
#pragma unroll
      for (int q = 0; q < MB; ++q) {  // 16-byte piece q of the row sits at q ^ i
        const double2 v = *reinterpret_cast<const double2*>(row + 2 * (q ^ i));
        if (2 * q < MB) {
          S[2 * q] = v.x;
          S[2 * q + 1] = v.y;
        } else {
          R[2 * q - MB] = v.x;
          R[2 * q - MB + 1] = v.y;
        }
      }
      if (WITH_F && act) fv = __ldg(g.f + (b0 + tt) * MB + i);
    }
    // Gauss-Jordan on [R | S | f]: pivot row k broadcast through PB as
    // 16-byte pairs (two alternating buffers: one __syncwarp per pivot)
    double dg = 1.0;
#pragma unroll
    for (int k = 0; k < MB; ++k) {
      double2* pb = reinterpret_cast<double2*>(PB + (k & 1) * C::PIV);
      if (i == k) {  // the pivot lane publishes its row and the pivot's reciprocal
#pragma unroll
        for (int c = 2 * (k / 2); c < MB; c += 2) pb[c / 2] = make_double2(R[c], R[c + 1]);
#pragma unroll
        for (int c = 0; c < MB; c += 2) pb[(MB + c) / 2] = make_double2(S[c], S[c + 1]);
        pb[MB] = make_double2(fv, fast_rcp(R[k]));
      }
      __syncwarp();
      double pr[MB], ps[MB];
#pragma unroll
      for (int c = 2 * (k / 2); c < MB; c += 2) {
        const double2 v = pb[c / 2];
        pr[c] = v.x;
        pr[c + 1] = v.y;
      }
#pragma unroll
      for (int c = 0; c < MB; c += 2) {
        const double2 v = pb[(MB + c) / 2];
        ps[c] = v.x;
        ps[c + 1] = v.y;
      }
      const double2 frp = pb[MB];
      // branch-free: the pivot lane applies a zero multiplier
      const bool me = i == k;
      dg = me ? pr[k] : dg;
      const double m = me ? 0.0 : R[k] * frp.y;
#pragma unroll
      for (int c = k + 1; c < MB; ++c) R[c] = fma(-m, pr[c], R[c]);
#pragma unroll
      for (int c = 0; c < MB; ++c) S[c] = fma(-m, ps[c], S[c]);
      if (WITH_F) fv = fma(-m, frp.x, fv);
    }
    const double rd = fast_rcp(dg);
    double T[MB];
#pragma unroll
    for (int c = 0; c < MB; ++c) T[c] = -S[c] * rd;
    const double ci = fv * rd;
    // this block's phi component: phi_i <- T_b[i] . phi + c_i (phi of the
    // previous block is in every lane)
    double phi_i = ci;
    if (WITH_F)
#pragma unroll
      for (int l = 0; l < MB; ++l) phi_i = fma(T[l], ph[l], phi_i);
    if (act) {
      if (STORE_T) {
        double2* dst = reinterpret_cast<double2*>(g.tm + (b0 + tt - 1) * MM) + i;
#pragma unroll
        for (int q = 0; q < MB / 2; ++q) dst[q * MB] = make_double2(T[2 * q], T[2 * q + 1]);
      }
      if (WITH_F) g.cv[(b0 + tt) * MB + i] = ci;
    }
    // publish T_b (row i) and phi_i, then fold the block into the chunk map
    double* TBk = TB;
#pragma unroll
    for (int c = 0; c < MB; c += 2) *reinterpret_cast<double2*>(TBk + i * C::TP + c) = make_double2(T[c], T[c + 1]);
    if (WITH_F) TBk[MB * C::TP + i] = phi_i;
    __syncwarp();
    if (act) {
      double np[MB];
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        double a = 0.0;
#pragma unroll
        for (int c = 0; c < MB; c += 2) {
          const double2 m = *reinterpret_cast<const double2*>(TBk + r * C::TP + c);
          a = fma(m.y, pc[c + 1], fma(m.x, pc[c], a));
        }
        np[r] = a;
      }
#pragma unroll
      for (int r = 0; r < MB; ++r) pc[r] = np[r];
      if (WITH_F)
#pragma unroll
        for (int r = 0; r < MB; r += 2) {
          const double2 v = *reinterpret_cast<const double2*>(TBk + MB * C::TP + r);
          ph[r] = v.x;
          ph[r + 1] = v.y;
        }
    }
    __syncwarp();  // TB is published again by the next block
  }
  cp_async_wait<0>();
  if (live) {
    if (STORE_T)
#pragma unroll
      for (int r = 0; r < MB; ++r) t.phi[0][j * MM + r * MB + i] = pc[r];
    if (WITH_F) {
      t.fl[1][(j + 1) * MB + i] = pick<MB>(ph, i);
      if (j == 0) t.fl[1][i] = __ldg(g.f + i);
    }
  }
  // ---- level 1: the CTA's 8 / MB level-1 chunks by a shared-memory tree
  const int T = t.T;
  const int gsub = wid * C::SG + sg;  // subgroup index in the CTA
  if (!live) {  // identity beyond the last chunk
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      pc[r] = r == i ? 1.0 : 0.0;
      ph[r] = 0.0;
    }
  }
  __syncthreads();
  fc_tree16<MB, WITH_F>(fsm, gsub, i, pc, ph);
  if (T == 1) {  // the level-0 maps were the top (one CTA)
    if (STORE_T && gsub == 0) chain_fc_top<MB>(g, t, fsm, lane, pc);
    return;
  }
  {
    const long c1 = (long)blockIdx.x * C::L1C + gsub / kChainC0;
    if (gsub % kChainC0 == 0 && c1 * kChainC0 < P0) {
      if (STORE_T)
#pragma unroll
        for (int r = 0; r < MB; ++r) t.phi[1][c1 * MM + r * MB + i] = pc[r];
      if (WITH_F) {
        t.fl[2][(c1 + 1) * MB + i] = pick<MB>(ph, i);
        if (c1 == 0) t.fl[2][i] = __ldg(g.f + i);
      }
    }
  }
  // ---- levels >= 2 and the top: the last arriving CTA composes (16 subgroups)
  long cprev = (long)blockIdx.x;  // arrival unit at level 2: this CTA
  for (int l = 2;; ++l) {
    const bool top = l == T;
    long cc;
    int expected, len;
    if (top) {
      cc = 0;
      expected = T == 2 ? (int)gridDim.x : t.P[T - 1];
      len = t.P[T - 1];
    } else {
      cc = l == 2 ? cprev * C::L1C / kChainC0 : cprev / kChainC0;
      if (l == 2) {
        const long first_cta = cc * kChainC0 / C::L1C;
        const long last_cta = min((long)gridDim.x, (cc + 1) * kChainC0 / C::L1C);
        expected = (int)(last_cta - first_cta);
      } else {
        expected = (int)min((long)kChainC0, (long)t.P[l - 1] - kChainC0 * cc);
      }
      len = (int)min((long)kChainC0, (long)t.P[l - 1] - kChainC0 * cc);
    }
    if (!cta_last_arrive(t.cnt + t.coff[l] + cc, expected)) return;
    const double* maps = t.phi[l - 1] + cc * kChainC0 * MM;
    const double* vecs = t.fl[l] + (cc * kChainC0 + 1) * MB;
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      const bool have = gsub < len;
      pc[r] = have ? __ldcg(maps + (long)gsub * MM + r * MB + i) : (r == i ? 1.0 : 0.0);
      ph[r] = have && WITH_F ? __ldcg(vecs + (long)gsub * MB + r) : 0.0;
    }
    fc_tree16<MB, WITH_F>(fsm, gsub, i, pc, ph);
    if (top) {
      if (STORE_T && gsub == 0) chain_fc_top<MB>(g, t, fsm, lane, pc);
      return;
    }
    if (gsub == 0) {
      if (STORE_T)
#pragma unroll
        for (int r = 0; r < MB; ++r) t.phi[l][cc * MM + r * MB + i] = pc[r];
      if (WITH_F) {
        t.fl[l + 1][(cc + 1) * MB + i] = pick<MB>(ph, i);
        if (cc == 0) t.fl[l + 1][i] = __ldg(g.f + i);
      }
    }
    cprev = cc;
  }
}

// ---------------------------------------------------------------------------
// chain_fc2_kernel (m = 8): chain_fc_kernel with TWO rows per lane -- MB / 2
// lanes per block, lane i = rows i and i + MB/2 of every block and columns i
// and i + MB/2 of Phi.  Same arithmetic, element by element, as
// chain_fc_kernel (bit-identical results).  The row-per-lane kernel is bound
// by the shared-memory data pipe (profiles/r02_ncu_full_cfg4.txt: 15 M load +
// 10 M store wavefronts, MIO throttle the first stall); what changes:
//  * the pivot row reaches the other lanes of its subgroup by shuffles (one
//    LSU wavefront each; the shared-memory broadcast cost ~4.5 wavefronts per
//    sparse 16-byte store plus the read-back, a divergent publish and a
//    __syncwarp per pivot), and it serves two rows per lane;
//  * the read-back of T_b for the composition serves two columns per lane;
//  * two shared regions with their own pitch per subgroup (rows: 64 bytes mod
//    128, T_b: 16 bytes mod 128), so neither the row reads nor the broadcast
//    reads of the 8 subgroups of a warp conflict;
//  * f one block ahead in registers, the next pivot's reciprocal started by
//    every lane as soon as its column is updated;
//  * CTAs of 16 chunks (one level-1 chunk, 2 warps): 1024 small CTAs balance
//    over the SMs where 512 large ones left a 30 % tail.
// Measured (config 4): 161 -> 122 us.  Not kept: the block by
// COLUMNS (pivot column = 8 values per pivot instead of 17, no swizzle, bulk
// copies: 15 M instead of 20 M wavefronts but 38 M instead of 31 M
// instructions and f / phi replicated: 155 us), rows by 128-byte bulk copies
// at a 144-byte pitch (183 us: the small copies and the mbarrier polls), one
// stage buffer for 6 CTAs per SM (126 us) or 7 with 128 registers (129 us:
// the SM's shared-memory pipe, not its occupancy, sets the pace; 4 CTAs per SM
// also spread the 1024 CTAs more evenly).
// ---------------------------------------------------------------------------
template <int MB>
struct Fc2Cfg {
  static constexpr int LPB = MB / 2;                                  // lanes per block (chunk)
  static constexpr int SG = 32 / LPB;                                 // subgroups (chunks) per warp
  static constexpr int NW = kChainC0 / SG;                            // warps per CTA: 16 chunks = one level-1 chunk
  static constexpr int CPC = NW * SG;                                 // level-0 chunks per CTA
  static constexpr int L1C = CPC / kChainC0;                          // level-1 chunks per CTA
  static constexpr int BLK = 2 * MB * MB;                             // [S | R] doubles per block row
  static constexpr int TP = MB + 2;                                   // row pitch of the published T_b
  static constexpr int TBS = MB * TP + MB;                            // published T_b + phi
  static constexpr int STG = ((2 * BLK + 15) / 16) * 16 + 8;          // stage pitch: 64 bytes mod 128
  static constexpr int SUB = ((TBS + 15) / 16) * 16 + 2;              // T_b pitch: 16 bytes mod 128
  static constexpr int NSUB = NW * SG;
  static constexpr int SMEM = NSUB * (STG + SUB) * 8;                 // bytes per CTA
};

// fc_tree16 for two columns per lane (pa: column i, pb: column i + MB/2)
template <int MB, bool VEC>
__device__ __forceinline__ void fc2_tree16(double* fsm, int gsub, int i, double (&pa)[MB], double (&pb)[MB],
                                           double (&ph)[MB]) {
  using C = Fc2Cfg<MB>;
  constexpr int H = C::LPB;
  const int s = gsub % kChainC0;
#pragma unroll 1
  for (int h = 1; h < kChainC0; h <<= 1) {
    double* mine = fsm + C::NSUB * C::STG + gsub * C::SUB;  // TB region: MB x TP, then MB for phi
    if (s % (2 * h) == h) {  // later partner of (s - h): publish
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        mine[r * C::TP + i] = pa[r];
        mine[r * C::TP + i + H] = pb[r];
      }
      if (VEC) {
        mine[MB * C::TP + i] = pick<MB>(ph, i);
        mine[MB * C::TP + i + H] = pick<MB>(ph, i + H);
      }
    }
    __syncthreads();
    if (s % (2 * h) == 0) {
      const double* L = fsm + C::NSUB * C::STG + (gsub + h) * C::SUB;
      double na[MB], nb[MB], nv[MB];
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        double a = 0.0, b = 0.0, v = VEC ? L[MB * C::TP + r] : 0.0;
#pragma unroll
        for (int c = 0; c < MB; c += 2) {
          const double2 m = *reinterpret_cast<const double2*>(L + r * C::TP + c);
          a = fma(m.y, pa[c + 1], fma(m.x, pa[c], a));
          b = fma(m.y, pb[c + 1], fma(m.x, pb[c], b));
          if (VEC) v = fma(m.y, ph[c + 1], fma(m.x, ph[c], v));
        }
        na[r] = a;
        nb[r] = b;
        nv[r] = v;
      }
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        pa[r] = na[r];
        pb[r] = nb[r];
        if (VEC) ph[r] = nv[r];
      }
    }
    __syncthreads();
  }
}

// chain_fc_top for the two-columns-per-lane layout: the whole of warp 0 calls
// it (pa / pb valid in lanes 0..MB/2-1).  G = Ba + Bb Phi_total is built in
// shared memory, then factored with lane i = row i (lanes >= MB replicate row
// lane % MB): every lane sees the pivot column by shuffles and runs the same
// first-maximum scan, the two rows change lanes by shuffles, the update is the
// serial algorithm's element by element (bit-identical LU; one lane working
// through shared memory took 9.3 us at the end of the factor launch).
template <int MB>
__device__ void chain_fc2_top(const ChainLevelArgs& g, const ChainTree& t, double* buf, int lane, const double (&pa)[MB],
                              const double (&pb)[MB]) {
  constexpr int MM = MB * MB, GP = MB + 1, H = MB / 2;
  if (lane < H) {
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      double va = __ldg(g.data + r * MB + lane), vb = __ldg(g.data + r * MB + lane + H);
#pragma unroll
      for (int l = 0; l < MB; ++l) {
        const double bb = __ldg(g.corner + r * MB + l);
        va = fma(bb, pa[l], va);
        vb = fma(bb, pb[l], vb);
      }
      buf[r * GP + lane] = va;
      buf[r * GP + lane + H] = vb;
    }
  }
  __syncwarp();
  TL_MAX(12, 0);
  const int i = lane % MB;
  double gr[MB];
#pragma unroll
  for (int c = 0; c < MB; ++c) gr[c] = buf[i * GP + c];
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    // partial pivoting: the first row >= k with the largest |G[r][k]|
    const double mine = fabs(gr[k]);
    int p = k;
    double best = gshfl<MB>(mine, k);
#pragma unroll
    for (int r = k + 1; r < MB; ++r) {
      const double v = gshfl<MB>(mine, r);
      if (v > best) {
        best = v;
        p = r;
      }
    }
    double pr[MB];
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      const double rk = gshfl<MB>(gr[c], k), rp = gshfl<MB>(gr[c], p);
      pr[c] = rp;  // the pivot row after the interchange
      gr[c] = i == k ? rp : (i == p ? rk : gr[c]);
    }
    if (lane == 0) t.glu[MM + k] = (double)p;
    if (i > k) {
      const double l = gr[k] / pr[k];
      gr[k] = l;
#pragma unroll
      for (int c = k + 1; c < MB; ++c) gr[c] = fma(-l, pr[c], gr[c]);
    }
  }
  TL_MAX(12, 1);
  if (lane < MB)
#pragma unroll
    for (int c = 0; c < MB; ++c) t.glu[i * MB + c] = gr[c];
  __syncwarp();
}

template <int MB, bool STORE_T, bool WITH_F>
__global__ void __launch_bounds__(Fc2Cfg<MB>::NW * 32) chain_fc2_kernel(ChainLevelArgs g, ChainTree t) {
  TL_MIN(0, 0);
  pdl_trigger();  // the down sweep may launch (it waits for this grid before reading anything)
  using C = Fc2Cfg<MB>;
  constexpr int MM = MB * MB, RW = 2 * MB, H = C::LPB, NP = RW / 2;  // NP 16-byte pieces per row
  extern __shared__ __align__(16) double fsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, sg = lane / H, i = lane % H;
  double* stage = fsm + (wid * C::SG + sg) * C::STG;                     // 2 x BLK
  double* TB = fsm + C::NSUB * C::STG + (wid * C::SG + sg) * C::SUB;    // MB x TP published T_b, then phi
  const long P0 = t.P[0];
  const long j = (long)blockIdx.x * C::CPC + wid * C::SG + sg;  // level-0 chunk
  const bool live = j < P0;
  const long nblk = (long)g.nb - 1;                             // blocks after the BC row
  const int len = live ? (int)min((long)kChainC0, nblk - kChainC0 * j) : 0;
  const long b0 = kChainC0 * j + 1;                             // first block row of the chunk
  // block row b0 + tt into stage buffer tt & 1: 16-byte cp.async pieces, piece
  // c of row q at c ^ q (lane i then reads its rows conflict-free)
  auto issue = [&](int tt) {
    if (tt < len) {
      const double* src = g.data + MM + (b0 + tt - 1) * C::BLK;
      double* dst = stage + (tt & 1) * C::BLK;
#pragma unroll
      for (int q = 0; q < MB; ++q)
#pragma unroll
        for (int hh = 0; hh < NP / H; ++hh) {
          const int c = hh * H + i;
          cp_async16(dst + q * RW + 2 * (c ^ q), src + q * RW + 2 * c);
        }
    }
    cp_async_commit();
  };
  double pa[MB], pq[MB], ph[MB];  // columns i and i + H of Phi, the whole phi
#pragma unroll
  for (int r = 0; r < MB; ++r) {
    pa[r] = r == i ? 1.0 : 0.0;
    pq[r] = r == i + H ? 1.0 : 0.0;
    ph[r] = 0.0;
  }
  issue(0);
  double fn0 = 0.0, fn1 = 0.0;  // f of the next block (one step ahead)
  if (WITH_F && len > 0) {
    fn0 = __ldg(g.f + b0 * MB + i);
    fn1 = __ldg(g.f + b0 * MB + i + H);
  }
#pragma unroll 1
  for (int tt = 0; tt < kChainC0; ++tt) {
    issue(tt + 1);
    cp_async_wait<1>();
    __syncwarp();
    const bool act = tt < len;
    double R0[MB], S0[MB], R1[MB], S1[MB], f0 = fn0, f1 = fn1;
    if (WITH_F) {
      const bool nx = tt + 1 < len;
      fn0 = nx ? __ldg(g.f + (b0 + tt + 1) * MB + i) : 0.0;
      fn1 = nx ? __ldg(g.f + (b0 + tt + 1) * MB + i + H) : 0.0;
    }
    {
      const double* row0 = stage + (tt & 1) * C::BLK + i * RW;
      const double* row1 = row0 + H * RW;
#pragma unroll
      for (int q = 0; q < NP; ++q) {  // 16-byte piece q of row r sits at q ^ r
        const double2 v = *reinterpret_cast<const double2*>(row0 + 2 * (q ^ i));
        const double2 w = *reinterpret_cast<const double2*>(row1 + 2 * (q ^ (i + H)));
        if (2 * q < MB) {
          S0[2 * q] = v.x;
          S0[2 * q + 1] = v.y;
          S1[2 * q] = w.x;
          S1[2 * q + 1] = w.y;
        } else {
          R0[2 * q - MB] = v.x;
          R0[2 * q - MB + 1] = v.y;
          R1[2 * q - MB] = w.x;
          R1[2 * q - MB + 1] = w.y;
        }
      }
    }
    // Gauss-Jordan on [R | S | f]; the next pivot's reciprocal is started by
    // every lane as soon as its column is updated
    double dg0 = 1.0, dg1 = 1.0;
    double rc = fast_rcp(R0[0]);
#pragma unroll
    for (int k = 0; k < MB; ++k) {
      // pivot row k lives in lane k % H (slot k / H): its entries reach the
      // other lanes of the subgroup by shuffles (one LSU wavefront each; the
      // shared-memory broadcast cost ~4.5 wavefronts per sparse 16-byte store
      // plus the read-back, and a divergent publish + __syncwarp per pivot)
      const bool own = i == k % H;
      double pr[MB], ps[MB];
#pragma unroll
      for (int c = k + 1; c < MB; ++c) pr[c] = gshfl<H>(k < H ? R0[c] : R1[c], k % H);
#pragma unroll
      for (int c = 0; c < MB; ++c) ps[c] = gshfl<H>(k < H ? S0[c] : S1[c], k % H);
      double2 frp;
      frp.x = WITH_F ? gshfl<H>(k < H ? f0 : f1, k % H) : 0.0;
      frp.y = gshfl<H>(rc, k % H);
      pr[k] = k < H ? R0[k] : R1[k];  // read by the pivot lane only (its own diagonal entry)
      // branch-free: the pivot row itself takes a zero multiplier
      const bool me0 = own && k < H, me1 = own && k >= H;
      dg0 = me0 ? pr[k] : dg0;
      dg1 = me1 ? pr[k] : dg1;
      const double m0 = me0 ? 0.0 : R0[k] * frp.y;
      const double m1 = me1 ? 0.0 : R1[k] * frp.y;
#pragma unroll
      for (int c = k + 1; c < MB; ++c) {
        R0[c] = fma(-m0, pr[c], R0[c]);
        R1[c] = fma(-m1, pr[c], R1[c]);
      }
      if (k + 1 < MB) rc = fast_rcp(k + 1 < H ? R0[k + 1] : R1[k + 1]);
#pragma unroll
      for (int c = 0; c < MB; ++c) {
        S0[c] = fma(-m0, ps[c], S0[c]);
        S1[c] = fma(-m1, ps[c], S1[c]);
      }
      if (WITH_F) {
        f0 = fma(-m0, frp.x, f0);
        f1 = fma(-m1, frp.x, f1);
      }
    }
    const double rd0 = fast_rcp(dg0), rd1 = fast_rcp(dg1);
#pragma unroll
    for (int c = 0; c < MB; ++c) {  // S becomes T_b = -D^-1 S'
      S0[c] = -S0[c] * rd0;
      S1[c] = -S1[c] * rd1;
    }
    const double ci0 = f0 * rd0, ci1 = f1 * rd1;
    // this block's phi components: phi_r <- T_b[r] . phi + c_r
    double phi0 = ci0, phi1 = ci1;
    if (WITH_F)
#pragma unroll
      for (int l = 0; l < MB; ++l) {
        phi0 = fma(S0[l], ph[l], phi0);
        phi1 = fma(S1[l], ph[l], phi1);
      }
    if (act) {
      if (STORE_T) {
        double2* dst = reinterpret_cast<double2*>(g.tm + (b0 + tt - 1) * MM) + i;
#pragma unroll
        for (int q = 0; q < MB / 2; ++q) {
          dst[q * MB] = make_double2(S0[2 * q], S0[2 * q + 1]);
          dst[q * MB + H] = make_double2(S1[2 * q], S1[2 * q + 1]);
        }
      }
      if (WITH_F) {
        g.cv[(b0 + tt) * MB + i] = ci0;
        g.cv[(b0 + tt) * MB + i + H] = ci1;
      }
    }
    // publish T_b (rows i, i + H) and phi, then fold the block into the chunk map
#pragma unroll
    for (int c = 0; c < MB; c += 2) {
      *reinterpret_cast<double2*>(TB + i * C::TP + c) = make_double2(S0[c], S0[c + 1]);
      *reinterpret_cast<double2*>(TB + (i + H) * C::TP + c) = make_double2(S1[c], S1[c + 1]);
    }
    if (WITH_F) {
      TB[MB * C::TP + i] = phi0;
      TB[MB * C::TP + i + H] = phi1;
    }
    __syncwarp();
    if (act) {
      double na[MB], nq[MB];
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int c = 0; c < MB; c += 2) {
          const double2 m = *reinterpret_cast<const double2*>(TB + r * C::TP + c);
          a = fma(m.y, pa[c + 1], fma(m.x, pa[c], a));
          b = fma(m.y, pq[c + 1], fma(m.x, pq[c], b));
        }
        na[r] = a;
        nq[r] = b;
      }
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        pa[r] = na[r];
        pq[r] = nq[r];
      }
      if (WITH_F)
#pragma unroll
        for (int r = 0; r < MB; r += 2) {
          const double2 v = *reinterpret_cast<const double2*>(TB + MB * C::TP + r);
          ph[r] = v.x;
          ph[r + 1] = v.y;
        }
    }
    __syncwarp();  // TB is published again by the next block
  }
  cp_async_wait<0>();
  if (live) {
    if (STORE_T)
#pragma unroll
      for (int r = 0; r < MB; ++r) {
        t.phi[0][j * MM + r * MB + i] = pa[r];
        t.phi[0][j * MM + r * MB + i + H] = pq[r];
      }
    if (WITH_F) {
      t.fl[1][(j + 1) * MB + i] = pick<MB>(ph, i);
      t.fl[1][(j + 1) * MB + i + H] = pick<MB>(ph, i + H);
      if (j == 0) {
        t.fl[1][i] = __ldg(g.f + i);
        t.fl[1][i + H] = __ldg(g.f + i + H);
      }
    }
  }
  // ---- level 1: the CTA's level-1 chunk by a shared-memory tree
  const int T = t.T;
  const int gsub = wid * C::SG + sg;  // subgroup index in the CTA
  if (!live) {  // identity beyond the last chunk
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      pa[r] = r == i ? 1.0 : 0.0;
      pq[r] = r == i + H ? 1.0 : 0.0;
      ph[r] = 0.0;
    }
  }
  __syncthreads();
  fc2_tree16<MB, WITH_F>(fsm, gsub, i, pa, pq, ph);
  if (T == 1) {  // the level-0 maps were the top (one CTA)
    if (STORE_T && threadIdx.x < 32) chain_fc2_top<MB>(g, t, fsm, lane, pa, pq);
    return;
  }
  {
    const long c1 = (long)blockIdx.x * C::L1C + gsub / kChainC0;
    if (gsub % kChainC0 == 0 && c1 * kChainC0 < P0) {
      if (STORE_T)
#pragma unroll
        for (int r = 0; r < MB; ++r) {
          t.phi[1][c1 * MM + r * MB + i] = pa[r];
          t.phi[1][c1 * MM + r * MB + i + H] = pq[r];
        }
      if (WITH_F) {
        t.fl[2][(c1 + 1) * MB + i] = pick<MB>(ph, i);
        t.fl[2][(c1 + 1) * MB + i + H] = pick<MB>(ph, i + H);
        if (c1 == 0) {
          t.fl[2][i] = __ldg(g.f + i);
          t.fl[2][i + H] = __ldg(g.f + i + H);
        }
      }
    }
  }
  TL_MAX(8, 0);
  // ---- levels >= 2 and the top: the last arriving CTA composes (16 subgroups)
  long cprev = (long)blockIdx.x;  // arrival unit at level 2: this CTA
  for (int l = 2;; ++l) {
    const bool top = l == T;
    long cc;
    int expected, len2;
    if (top) {
      cc = 0;
      expected = T == 2 ? (int)gridDim.x : t.P[T - 1];
      len2 = t.P[T - 1];
    } else {
      cc = l == 2 ? cprev * C::L1C / kChainC0 : cprev / kChainC0;
      if (l == 2) {
        const long first_cta = cc * kChainC0 / C::L1C;
        const long last_cta = min((long)gridDim.x, (cc + 1) * kChainC0 / C::L1C);
        expected = (int)(last_cta - first_cta);
      } else {
        expected = (int)min((long)kChainC0, (long)t.P[l - 1] - kChainC0 * cc);
      }
      len2 = (int)min((long)kChainC0, (long)t.P[l - 1] - kChainC0 * cc);
    }
    if (!cta_last_arrive(t.cnt + t.coff[l] + cc, expected)) return;
    TL_MAX(7 + l, 1);
    const double* maps = t.phi[l - 1] + cc * kChainC0 * MM;
    const double* vecs = t.fl[l] + (cc * kChainC0 + 1) * MB;
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      const bool have = gsub < len2;
      pa[r] = have ? __ldcg(maps + (long)gsub * MM + r * MB + i) : (r == i ? 1.0 : 0.0);
      pq[r] = have ? __ldcg(maps + (long)gsub * MM + r * MB + i + H) : (r == i + H ? 1.0 : 0.0);
      ph[r] = have && WITH_F ? __ldcg(vecs + (long)gsub * MB + r) : 0.0;
    }
    fc2_tree16<MB, WITH_F>(fsm, gsub, i, pa, pq, ph);
    TL_MAX(7 + l, 3);
    if (top) {
      if (STORE_T && threadIdx.x < 32) chain_fc2_top<MB>(g, t, fsm, lane, pa, pq);
      TL_MAX(0, 1);
      return;
    }
    if (gsub == 0) {
      if (STORE_T)
#pragma unroll
        for (int r = 0; r < MB; ++r) {
          t.phi[l][cc * MM + r * MB + i] = pa[r];
          t.phi[l][cc * MM + r * MB + i + H] = pq[r];
        }
      if (WITH_F) {
        t.fl[l + 1][(cc + 1) * MB + i] = pick<MB>(ph, i);
        t.fl[l + 1][(cc + 1) * MB + i + H] = pick<MB>(ph, i + H);
        if (cc == 0) {
          t.fl[l + 1][i] = __ldg(g.f + i);
          t.fl[l + 1][i + H] = __ldg(g.f + i + H);
        }
      }
    }
    cprev = cc;
  }
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
#ifndef PSG_CS_PRE1
#define PSG_CS_PRE1 2
#endif
#ifndef PSG_CS_PRE2
#define PSG_CS_PRE2 2
#endif
#ifndef PSG_CS_MINB1
#define PSG_CS_MINB1 7
#endif
#ifndef PSG_CS_MINB2
#define PSG_CS_MINB2 7
#endif
// ring depth / resident CTAs per SM asked for, per pass (MODE 0 condense, 1 final, 2 correction).
// 2 deep at 72 registers = 7 CTAs of 128 threads per SM: all 1024 CTAs of config 4
// resident in one wave (3 deep at 96 registers = 5 per SM left a second wave of
// 284 CTAs running at a fraction of the bandwidth).
constexpr int chain_pre(int mode) { return mode == 2 ? PSG_CS_PRE2 : PSG_CS_PRE1; }
constexpr int chain_minb(int mode) { return mode == 2 ? PSG_CS_MINB2 : PSG_CS_MINB1; }

template <int MB>
struct ChainReg {  // staged maps (padded rows: conflict-free) + rhs slots of one <= 16-step chain
  static constexpr int MP = MB + 1;
  static constexpr int MAPS = kChainC0 * MB * MP;
  static constexpr int SIZE = MAPS + (kChainC0 + 1) * MB;
};

// maps[first + s] (s < len) and rhs[rfirst + s] (s < nr); cooperative over nthr threads.
// Every element goes global -> shared by an 8-byte cp.async (no register round
// trip: all of a thread's copies are in flight at once; the plain load + store
// loop waited for each batch of loads, and the long-scoreboard stalls were most of
// the down sweep's life); the coherent rhs (values another CTA of this grid
// wrote) keeps its ld.cg.  chain_stage_wait() before the barrier that
// publishes the region.
template <int MB>
__device__ __forceinline__ void chain_stage_maps(double* reg, const double* maps, long first, int len, int tid,
                                                 int nthr) {
  constexpr int MM = MB * MB, MP = MB + 1;
  const double* src = maps + first * MM;
  if (nthr % MM == 0 || MM % nthr == 0) {
    // a thread's elements sit at fixed (row, column) positions: no per-element division
    if (nthr >= MM) {  // nthr / MM maps per round, one element each
      const int r = tid % MM, ds = nthr / MM;
      double* dst = reg + (r / MB) * MP + r % MB;
      for (int s = tid / MM; s < len; s += ds) cp_async8(dst + s * MB * MP, src + s * MM + r);
    } else {           // MM / nthr elements of every map
      for (int s = 0; s < len; ++s)
        for (int r = tid; r < MM; r += nthr) cp_async8(reg + s * MB * MP + (r / MB) * MP + r % MB, src + s * MM + r);
    }
    return;
  }
  for (int e = tid; e < len * MM; e += nthr) {
    const int s = e / MM, r = e % MM;
    cp_async8(reg + s * MB * MP + (r / MB) * MP + r % MB, src + e);
  }
}
template <int MB, bool COHERENT_RHS>
__device__ __forceinline__ void chain_stage_rhs(double* reg, const double* rhs, long rfirst, int nr, int tid,
                                                int nthr) {
  double* rr = reg + ChainReg<MB>::MAPS;
  for (int e = tid; e < nr * MB; e += nthr) {
    if (COHERENT_RHS)
      rr[e] = __ldcg(rhs + rfirst * MB + e);
    else
      cp_async8(rr + e, rhs + rfirst * MB + e);
  }
}
template <int MB, bool COHERENT_RHS>
__device__ __forceinline__ void chain_stage(double* reg, const double* maps, long first, int len, const double* rhs,
                                            long rfirst, int nr, int tid, int nthr) {
  chain_stage_maps<MB>(reg, maps, first, len, tid, nthr);
  chain_stage_rhs<MB, COHERENT_RHS>(reg, rhs, rfirst, nr, tid, nthr);
}
__device__ __forceinline__ void chain_stage_wait() { cp_async_wait_all(); }

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
  static constexpr int kPre = chain_pre(MODE);
  long b0 = 0;
  int len = 0;
  double Tq[kPre][MB], Cq[kPre], Xq[kPre];  // row i of T_b, c_b[i] (final) or x_b[i] (correction)

  __device__ __forceinline__ void fetch(const ChainLevelArgs& g, int i, int t, int slot) {
    constexpr int MM = MB * MB;
    if (t < len) {
      const double2* row = reinterpret_cast<const double2*>(g.tm + (b0 + t - 1) * MM) + i;
#pragma unroll
      for (int c = 0; c < MB / 2; ++c) {
        const double2 tv = __ldg(row + c * MB);
        Tq[slot][2 * c] = tv.x;
        Tq[slot][2 * c + 1] = tv.y;
      }
      if (MODE != 2)
        Cq[slot] = __ldg(g.cv + (b0 + t) * MB + i);
      else
        Xq[slot] = g.x[(b0 + t) * MB + i];
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
    double ytp = yts;  // MODE 2: the corrected x one block before the separator row
    if (MODE != 0 && live && j == 0) g.x[i] = yt;
#pragma unroll
    for (int t = 0; t < kChainC0; ++t) {
      const int sl = t % kPre;
      const bool act = t < len, last = t == len - 1;
      double a = MODE != 2 ? Cq[sl] : 0.0;
#pragma unroll
      for (int l = 0; l < MB; ++l) a = fma(Tq[sl][l], gshfl<MB>(y, l), a);
      const double xold = MODE == 2 ? Xq[sl] : 0.0;
      if (act) {
        const long os = (b0 + t) * MB + i;
        if (MODE == 2) ytp = yt;
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
    }
    if (MODE == 2) {
      // certificate of the corrected separator row (the chunk's last block row):
      // r = f - S x_prev - R x_sep, S terms first, then R terms (every group runs the shuffles)
      const bool cert_here = len > 0;
      double S[MB], R[MB];
      if (cert_here) load_row<MB>(g.data, b0 + len - 1, i, S, R);
      double sg = 0.0, ab = 0.0;
#pragma unroll
      for (int l = 0; l < MB; ++l) {
        const double pl = gshfl<MB>(ytp, l);
        if (cert_here) {
          const double p1 = S[l] * pl;
          sg += p1;
          ab += fabs(p1);
        }
      }
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
        const double fv = __ldg(g.f + (b0 + len - 1) * MB + i);
        const double on = fabs(fv - sg), od = fabs(fv) + ab;
        if (on * den > num * od || (den == 0.0 && on > 0)) {
          num = on;
          den = od;
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
    chain_stage_wait();
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
__device__ void chain_top_solve(const ChainTree& t, const double (&bb)[MB], const double* regT,
                                const double* s_glu, double* s_r, double* s_top, int lane) {
  constexpr int MM = MB * MB;
  const int i = lane % MB, PT = t.P[t.T - 1];
  const double* rT = regT + ChainReg<MB>::MAPS;
  double y = chain_condense<MB>(regT, PT, i);
  double r = rT[i];
#pragma unroll
  for (int l = 0; l < MB; ++l) r = fma(-bb[l], gshfl<MB>(y, l), r);
  // stored LU of G (row interchanges, unit lower, upper): lane i = row i, the
  // right-hand side one component per lane, pivot values by shuffles (8
  // dependent steps per sweep; one lane working through shared memory took
  // ~2.5 us of each down sweep).  Forward sweep in the serial order; the
  // backward sweep is column-oriented (row i accumulates from column MB-1 down).
  double lu[MB];
#pragma unroll
  for (int l = 0; l < MB; ++l) lu[l] = s_glu[i * MB + l];
  const double dg = pick<MB>(lu, i);
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    const int p = (int)s_glu[MM + k];
    const double rk = gshfl<MB>(r, k), rp = gshfl<MB>(r, p);
    r = i == k ? rp : (i == p ? rk : r);
  }
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    const double rk = gshfl<MB>(r, k);
    if (i > k) r = fma(-lu[k], rk, r);
  }
  y = r;
#pragma unroll
  for (int k = MB - 1; k >= 0; --k) {
    const double q = r / dg;
    const double xk = gshfl<MB>(q, k);
    if (i == k) y = q;
    if (i < k) r = fma(-lu[k], xk, r);
  }
  (void)s_r;
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
  // launched programmatically: wait for the producer of F (and, sel 0, of the
  // maps), then let the next level-0 pass start its prologue (it waits on this
  // grid before reading the values written here).  The correction sweep
  // (sel 1) follows the final pass: its maps and the top LU date from the
  // factor launch, complete before the final pass started, so they are staged
  // while the final pass drains.
  // regions: top at ssm, level l (2 <= l < T) at ssm + (T - l) * REG
  auto stage = [&](bool maps, bool rhs) {
    if (maps) chain_stage_maps<MB>(ssm, t.phi[T - 1], 0, PT, lane, 32);
    if (rhs) chain_stage_rhs<MB, false>(ssm, F[T], 0, PT + 1, lane, 32);
    for (int l = 2; l < T; ++l) {
      const long cc = w >> (4 * (l - 2));
      const int len = (int)min((long)kChainC0, t.P[l - 1] - kChainC0 * cc);
      double* reg = ssm + (T - l) * REG;
      if (maps) chain_stage_maps<MB>(reg, t.phi[l - 1], kChainC0 * cc, len, lane, 32);
      if (rhs) chain_stage_rhs<MB, false>(reg, F[l], kChainC0 * cc, len + 1, lane, 32);
    }
    if (maps)
      for (int e = lane; e < MM + MB; e += 32) cp_async8(s_glu + e, t.glu + e);
  };
  double bb[MB];  // row i of Bb (user input: loaded ahead of the dependency wait)
#pragma unroll
  for (int l = 0; l < MB; ++l) bb[l] = __ldg(g.corner + i * MB + l);
  if (sel) stage(true, false);
  pdl_wait();
  TL_MIN(1 + 2 * sel, 0);
  // the correction sweep resets the status slot its successor (the correction
  // pass, the only kernel of a solve that reports) accumulates into
  if (sel && g.status && w == 0 && lane == 0) status_reset(g.status);
  // No early trigger: the next level-0 pass launches when this grid has
  // completed.  Letting its ~740 CTAs start their prologue (maps and ring
  // prefetch, ~25 MB of requests at once) beside the sweep filled the SMs'
  // load/store queues, and this latency-bound warp's shared loads and shuffles
  // waited behind them: 13-17 us per sweep against ~6 us alone (%globaltimer
  // stamps), config 4 0.261 -> 0.253 ms/step without the overlap.
  stage(!sel, true);
  chain_stage_wait();
  __syncwarp();
  TL_MAX(6 + sel, 0);
  chain_top_solve<MB>(t, bb, ssm, s_glu, s_r, s_top, lane);
  TL_MAX(6 + sel, 1);
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
  TL_MAX(6 + sel, 2);
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
  TL_MAX(1 + 2 * sel, 1);
}

// -DPSG_PROF: %globaltimer stamps of every CTA's phases (tools/prof_cs.py)
#ifdef PSG_PROF
__device__ long long g_prof[2][1024][6];
__device__ __forceinline__ long long gtime() {
  long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#define PSG_STAMP(k) \
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_prof[KM - 1][blockIdx.x][k] = gtime()
#else
#define PSG_STAMP(k)
#endif

template <int MB, int KM>
__global__ void __launch_bounds__(16 * MB, chain_minb(KM)) chain_solve_kernel(ChainLevelArgs g, ChainTree t) {
  PSG_STAMP(0);
  TL_MIN(2 * KM, 0);
  pdl_trigger();  // the next down sweep waits for this grid before reading anything it writes
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

  {
    constexpr int SEL = KM == 1 ? 0 : 1;
    double* const* Fd = SEL ? t.cfl : t.fl;  // rhs of the level-1 chain
    Pass0<MB, KM> ps;
    // the level-1 maps first: warp 0's walk needs them before anyone needs the ring
    // (maps ahead of the ring 0.2402 -> 0.2378 ms, ring after the maps landed -> 0.2369)
    if (T >= 2) chain_stage<MB, false>(reg1, t.phi[0], kChainC0 * c, len1, Fd[1], kChainC0 * c, len1 + 1, tid, NT);
    if (KM == 2)
      for (int e = tid; e < (len1 + 1) * MB; e += NT) s_x[e] = __ldg(t.x1 + kChainC0 * c * MB + e);
    chain_stage_wait();
    __syncthreads();
    ps.start(g, j, live, i);  // the ring's first loads travel while warp 0 walks the level-1 chain
    PSG_STAMP(1);
    if (tid < 32) {  // this CTA's level-1 values from the down sweep's level-2 values
      pdl_wait();  // launched programmatically after the down sweep: its values from here on
      TL_MIN(2 * KM, 2);
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
    PSG_STAMP(2);
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
      PSG_STAMP(3);
      if (tid < 32) chain_up<MB>(t, t.cfl, reg1, c, len1, lane);
      PSG_STAMP(4);
      TL_MAX(2 * KM, 1);
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
      PSG_STAMP(3);
      if (!finite) num = __longlong_as_double(0x7ff0000000000000ll), den = 1.0;
      if (g.status) cert_push(g.status, num, den);
      if (g.status && g.host_out) status_publish_last(g.status, g.host_out, g.done_ctr);
      PSG_STAMP(4);
      TL_MAX(2 * KM, 1);
    }
  }
}

}  // namespace psg
