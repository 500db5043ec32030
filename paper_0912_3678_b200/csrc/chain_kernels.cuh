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
//   factor  chain_tm_kernel: per block T_b and M_b = R_b^-1 (one block per
//           lane, LU in registers), stored beside the data; Phi_j by a
//           shared-memory tree product; the next level's rows [-Phi_j | I].
//   solve   chain_pass_kernel<0>: phi_j (condense) -> the reduced system in
//           x_sigma is again a BVP-layout BABD (S = -Phi, R = I, same Ba / Bb),
//           solved by the same kernels level by level, the last level by one
//           warp (chain_direct_kernel, partial pivoting on the BC system);
//           chain_pass_kernel<1>: x through every chunk from x_sigma, plus
//           the separator rows' residuals condensed to R^-1 r (the chain's
//           end value differs from the affine map by rounding, ~8 eps |x| per
//           step); one correction A d = r through the reduced levels and
//           chain_pass_kernel<2>: x += the homogeneous chain of d, certifying
//           the corrected separator rows (componentwise backward error),
//           chain_bc_cert_kernel the BC row.
//
// Passes: MB lanes per chunk (lane i = row i of every block), 32 / MB chunks
// per warp; shuffles are executed by the whole warp (shorter chunks idle).
#pragma once

#include "psg_common.cuh"

namespace psg {

// BVP-layout level: data = [Ba (MB*MB) | rows b = 1..nb-1: S_b | R_b (MB x 2MB, row-major)]
struct ChainLevelArgs {
  const double* data;
  const double* corner;  // Bb (MB x MB)
  int nb;                // block rows
  int P;                 // chunks
  const int* cut;        // P + 1 separator blocks: cut[0] = 0 .. cut[P] = nb - 1
  const double* f;       // rhs of this level (nb * MB)
  double* x;             // solution of this level (final pass)
  double* next_data;     // factor: next level's data ((P + 1) block rows)
  double* next_f;        // condense: next level's rhs
  const double* next_x;  // final: next level's solution (x at the separators)
  double* corr_f;        // final (optional): condensed separator residuals R_sep^-1 r_sep -> next level rhs
  double* tm;            // factor output / solve input: per block [T row i | M row i] (T = -R^-1 S, M = R^-1)
  int accumulate;        // final: x += chain of corr_x with zero forcing (the correction pass)
  const double* corr_x;  // accumulate: correction d at the separators (next_x keeps x_sep)
  DevStatus* status;
};

template <int MB>
__device__ __forceinline__ double gshfl(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src, MB);
}

// Solve R y = w in place on the row-per-lane layout (no pivoting, like the
// reference's Lu strategy): r[] = row `i` of R, w[] = NR right-hand sides.
template <int MB, int NR>
__device__ __forceinline__ void lane_solve(double (&r)[MB], double (&w)[NR], int i) {
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    const double pk = gshfl<MB>(r[k], k);
    const double l = r[k] * fast_rcp(pk);
#pragma unroll
    for (int c = k + 1; c < MB; ++c) {
      const double rk = gshfl<MB>(r[c], k);
      if (i > k) r[c] = fma(-l, rk, r[c]);
    }
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      const double wk = gshfl<MB>(w[c], k);
      if (i > k) w[c] = fma(-l, wk, w[c]);
    }
  }
  // back substitution, row k broadcast once solved
#pragma unroll
  for (int k = MB - 1; k >= 0; --k) {
    const double inv = fast_rcp(r[k]);
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      const double yk = gshfl<MB>(w[c] * inv, k);
      if (i == k) w[c] = yk;
      if (i < k) w[c] = fma(-r[k], yk, w[c]);
    }
  }
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

// factor: Phi_j, written as next level row j+1 = [ -Phi_j | I ]; chunk 0 also copies Ba.
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

template <int MB>
__global__ void __launch_bounds__(64) chain_tm_kernel(ChainLevelArgs g) {
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
  // ---- per lane: LU of R (no pivoting), then T = -R^-1 S and M = R^-1 column by column
  double* slot = sm + lane * SLOT;
  if (lane < nblk) {
    double R[MB * MB];
#pragma unroll
    for (int i = 0; i < MB; ++i)
#pragma unroll
      for (int c = 0; c < MB; ++c) R[(i) * MB + (c)] = slot[i * RW + MB + c];
#pragma unroll
    for (int k = 0; k < MB; ++k) {
      const double p = fast_rcp(R[k * MB + k]);
      R[k * MB + k] = p;  // keep the reciprocal pivot
#pragma unroll
      for (int i = 0; i < MB; ++i) {
        if (i > k) {
          const double l = R[i * MB + k] * p;
          R[i * MB + k] = l;
#pragma unroll
          for (int c = 0; c < MB; ++c)
            if (c > k) R[i * MB + c] = fma(-l, R[k * MB + c], R[i * MB + c]);
        }
      }
    }
#pragma unroll 1
    for (int c = 0; c < 2 * MB; ++c) {
      double y[MB];
#pragma unroll
      for (int i = 0; i < MB; ++i) y[i] = c < MB ? -slot[i * RW + c] : (i == c - MB ? 1.0 : 0.0);
#pragma unroll
      for (int i = 0; i < MB; ++i)
#pragma unroll
        for (int k = 0; k < MB; ++k)
          if (k < i) y[i] = fma(-R[i * MB + k], y[k], y[i]);
#pragma unroll
      for (int ii = 0; ii < MB; ++ii) {
        const int i = MB - 1 - ii;
#pragma unroll
        for (int k = 0; k < MB; ++k)
          if (k > i) y[i] = fma(-R[i * MB + k], y[k], y[i]);
        y[i] *= R[i * MB + i];
      }
#pragma unroll
      for (int i = 0; i < MB; ++i) slot[i * RW + c] = y[i];  // T (c < MB) over S, M over R
    }
  } else {  // missing blocks of a short last chunk: T = I
#pragma unroll
    for (int i = 0; i < MB; ++i)
#pragma unroll
      for (int c = 0; c < MB; ++c) slot[i * RW + c] = i == c ? 1.0 : 0.0;
  }
  __syncwarp();
  // ---- store [T | M] (same layout as the data rows)
  {
    double2* dst = reinterpret_cast<double2*>(g.tm + (bfirst - 1) * BW);
    const int tot2 = nblk * BW / 2;
    for (int e0 = lane; e0 < tot2; e0 += 32) {
      const int e = 2 * e0;
      dst[e0] = *reinterpret_cast<const double2*>(sm + (e / BW) * SLOT + e % BW);
    }
  }
  __syncwarp();
  // ---- Phi of the two chunks: tree of products P = later * earlier, in the T slots
#pragma unroll 1
  for (int h = 1; h < kChainC0; h <<= 1) {
    const int pairs = kChainC0 / (2 * h);  // per chunk
    if (lane < 2 * pairs) {
      const int c = lane / pairs, k = lane % pairs;
      double* Bs = sm + (c * kChainC0 + 2 * k * h) * SLOT;  // earlier (right factor), result slot
      const double* As = sm + (c * kChainC0 + 2 * k * h + h) * SLOT;
      double B[MB * MB];
#pragma unroll
      for (int i = 0; i < MB; ++i)
#pragma unroll
        for (int l = 0; l < MB; ++l) B[(i) * MB + (l)] = Bs[i * RW + l];
#pragma unroll
      for (int i = 0; i < MB; ++i) {
        double a[MB], o[MB];
#pragma unroll
        for (int l = 0; l < MB; ++l) a[l] = As[i * RW + l];
#pragma unroll
        for (int cc = 0; cc < MB; ++cc) {
          double acc = a[0] * B[(0) * MB + (cc)];
#pragma unroll
          for (int l = 1; l < MB; ++l) acc = fma(a[l], B[(l) * MB + (cc)], acc);
          o[cc] = acc;
        }
#pragma unroll
        for (int cc = 0; cc < MB; ++cc) Bs[i * RW + cc] = o[cc];
      }
    }
    __syncwarp();
  }
  // ---- next level rows: [ -Phi_j | I ] for the chunks of this warp
  for (int e = lane; e < 2 * BW; e += 32) {
    const int c = e / BW, r = e % BW, i = r / RW, cc = r % RW;
    const long j = 2 * w + c;
    if (j < g.P) {
      const double v = cc < MB ? -sm[c * kChainC0 * SLOT + i * RW + cc] : (i == cc - MB ? 1.0 : 0.0);
      g.next_data[MB * MB + j * BW + r] = v;
    }
  }
  if (w == 0)
    for (int e = lane; e < MB * MB; e += 32) g.next_data[e] = __ldg(g.data + e);
}

// ---------------------------------------------------------------------------
// chain passes: MB lanes per chunk (lane i = row i), 32 / MB chunks per warp.
// Each step needs row i of [T | M] (128 B per lane, 1 KB contiguous per
// group: coalesced) and f of the block; loads run kPre steps ahead in a
// register ring inside a fully unrolled kChainC0-step chain.  MODE 0:
// condense (phi, chain from zero), 1: final (x from x_sep, condensed
// separator residuals), 2: the correction (x += homogeneous chain of d,
// certificate of the corrected separator rows).  Chunk j = blocks
// 16j+1 .. 16j+16 (the last one may be shorter).
// ---------------------------------------------------------------------------
constexpr int kPre = 3;

template <int MB, int MODE>
__global__ void __launch_bounds__(128) chain_pass_kernel(ChainLevelArgs g) {
  constexpr int BW = 2 * MB * MB, RW = 2 * MB;
  const int lane = threadIdx.x & 31, i = lane % MB;
  const long j = ((long)blockIdx.x * blockDim.x + threadIdx.x) / MB;
  const bool live = j < g.P;
  const long b0 = live ? g.cut[j] + 1 : 1, b1 = live ? g.cut[j + 1] : 0;
  const int len = (int)(b1 - b0 + 1);
  double y = 0.0, yt = 0.0;
  if (MODE == 1 && live) y = yt = __ldg(g.next_x + j * MB + i);
  if (MODE == 2 && live) {
    y = __ldg(g.corr_x + j * MB + i);
    yt = __ldg(g.next_x + j * MB + i) + y;
  }
  if (MODE != 0 && live && j == 0) g.x[i] = yt;
  // register ring: T row, M row, f of the block (MODE 0/1), old x (MODE 2)
  double Tq[kPre][MB], Mq[kPre][MB], Fq[kPre][MB], Xq[kPre];
  auto fetch = [&](int t, int slot) {
    if (t < len) {
      const double2* row = reinterpret_cast<const double2*>(g.tm + (b0 + t - 1) * BW + (long)i * RW);
#pragma unroll
      for (int c = 0; c < MB / 2; ++c) {
        const double2 tv = __ldg(row + c);
        Tq[slot][2 * c] = tv.x;
        Tq[slot][2 * c + 1] = tv.y;
      }
      if (MODE != 2) {
        const double2* fr = reinterpret_cast<const double2*>(g.f + (b0 + t) * MB);
#pragma unroll
        for (int c = 0; c < MB / 2; ++c) {
          const double2 mv = __ldg(row + MB / 2 + c), fv = __ldg(fr + c);
          Mq[slot][2 * c] = mv.x;
          Mq[slot][2 * c + 1] = mv.y;
          Fq[slot][2 * c] = fv.x;
          Fq[slot][2 * c + 1] = fv.y;
        }
      } else {
        Xq[slot] = g.x[(b0 + t) * MB + i];
      }
    }
  };
#pragma unroll
  for (int t = 0; t < kPre; ++t) fetch(t, t);
  double num = 0.0, den = 0.0;
  bool finite = true;
#pragma unroll
  for (int t = 0; t < kChainC0; ++t) {
    const int sl = t % kPre;
    const bool act = t < len, last = t == len - 1;
    double a = 0.0;
    if (MODE != 2)
#pragma unroll
      for (int l = 0; l < MB; ++l) a = fma(Mq[sl][l], Fq[sl][l], a);
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
        const double xs = __ldg(g.next_x + (j + 1) * MB + i);
        if (g.corr_f) g.corr_f[(j + 1) * MB + i] = a - xs;  // R^-1 r_sep
        y = yt = xs;
      } else if (MODE == 2) {
        y = __ldg(g.corr_x + (j + 1) * MB + i);
        yt = __ldg(g.next_x + (j + 1) * MB + i) + y;
      } else {
        y = a;
      }
      if (MODE != 0) {
        g.x[os] = yt;
        finite &= isfinite(yt);
      }
    }
    if (t + kPre < kChainC0) fetch(t + kPre, sl);
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
  if (MODE == 0 && live) {
    g.next_f[(j + 1) * MB + i] = y;
    if (j == 0) g.next_f[i] = __ldg(g.f + i);
  }
  if (MODE == 1 && g.corr_f) {  // BC row residual (chunk 0; every group runs the shuffles)
    const bool bc = live && j == 0;
    const double x0 = bc ? __ldg(g.next_x + i) : 0.0;
    const double xe = bc ? __ldg(g.next_x + (long)g.P * MB + i) : 0.0;
    double sg = 0.0;
#pragma unroll
    for (int l = 0; l < MB; ++l) {
      const double a0 = gshfl<MB>(x0, l), ae = gshfl<MB>(xe, l);
      if (bc) sg += __ldg(g.data + i * MB + l) * a0 + __ldg(g.corner + i * MB + l) * ae;
    }
    if (bc) g.corr_f[i] = __ldg(g.f + i) - sg;
  }
  if (MODE != 0) {
    if (!finite) num = __longlong_as_double(0x7ff0000000000000ll), den = 1.0;
    if (g.status) cert_push(g.status, num, den);
  }
}

template <int MB>
__global__ void chain_bc_cert_kernel(ChainLevelArgs g) {
  const int lane = threadIdx.x, i = lane % MB;
  const double x0 = g.x[i], xe = g.x[(long)(g.nb - 1) * MB + i];
  double sg = 0.0, ab = 0.0;
#pragma unroll
  for (int l = 0; l < MB; ++l) {
    const double p1 = __ldg(g.data + i * MB + l) * gshfl<MB>(x0, l);
    const double p2 = __ldg(g.corner + i * MB + l) * gshfl<MB>(xe, l);
    sg += p1 + p2;
    ab += fabs(p1) + fabs(p2);
  }
  const double fv = __ldg(g.f + i);
  cert_push(g.status, fabs(fv - sg), fabs(fv) + ab);
}

// direct: the whole (small) level by one group of MB lanes: Phi = prod T_b,
// phi = chain from zero, (Ba + Bb Phi) x_0 = f_0 - Bb phi with partial
// pivoting, then the chain for x.
template <int MB>
__global__ void __launch_bounds__(32) chain_direct_kernel(ChainLevelArgs g) {
  const int lane = threadIdx.x, i = lane % MB;
  double phi[MB], ph = 0.0;
#pragma unroll
  for (int c = 0; c < MB; ++c) phi[c] = i == c ? 1.0 : 0.0;
  for (int b = 1; b < g.nb; ++b) {
    double S[MB], R[MB], w[MB + 1];
    load_row<MB>(g.data, b, i, S, R);
#pragma unroll
    for (int c = 0; c <= MB; ++c) w[c] = 0.0;
    w[MB] = __ldg(g.f + (long)b * MB + i);
#pragma unroll
    for (int l = 0; l < MB; ++l) {
#pragma unroll
      for (int c = 0; c < MB; ++c) w[c] = fma(-S[l], gshfl<MB>(phi[c], l), w[c]);
      w[MB] = fma(-S[l], gshfl<MB>(ph, l), w[MB]);
    }
    lane_solve<MB, MB + 1>(R, w, i);
#pragma unroll
    for (int c = 0; c < MB; ++c) phi[c] = w[c];
    ph = w[MB];
  }
  // M0 = Ba + Bb Phi, rhs = f_0 - Bb phi  (row i)
  double M0[MB], rhs = __ldg(g.f + i);
#pragma unroll
  for (int c = 0; c < MB; ++c) M0[c] = __ldg(g.data + i * MB + c);
#pragma unroll
  for (int l = 0; l < MB; ++l) {
    const double bb = __ldg(g.corner + i * MB + l);
#pragma unroll
    for (int c = 0; c < MB; ++c) M0[c] = fma(bb, gshfl<MB>(phi[c], l), M0[c]);
    rhs = fma(-bb, gshfl<MB>(ph, l), rhs);
  }
  // the small BC system: serial Gaussian elimination with partial pivoting on lane 0
  __shared__ double Msh[MB][MB + 1];
  if (lane < MB) {
#pragma unroll
    for (int c = 0; c < MB; ++c) Msh[i][c] = M0[c];
    Msh[i][MB] = rhs;
  }
  __syncwarp();
  if (lane == 0) {
    for (int k = 0; k < MB; ++k) {
      int p = k;
      for (int r2 = k + 1; r2 < MB; ++r2)
        if (fabs(Msh[r2][k]) > fabs(Msh[p][k])) p = r2;
      if (p != k)
        for (int c = 0; c <= MB; ++c) {
          const double t = Msh[k][c];
          Msh[k][c] = Msh[p][c];
          Msh[p][c] = t;
        }
      for (int r2 = k + 1; r2 < MB; ++r2) {
        const double l = Msh[r2][k] / Msh[k][k];
        for (int c = k; c <= MB; ++c) Msh[r2][c] = fma(-l, Msh[k][c], Msh[r2][c]);
      }
    }
    for (int k = MB - 1; k >= 0; --k) {
      double s = Msh[k][MB];
      for (int c = k + 1; c < MB; ++c) s = fma(-Msh[k][c], Msh[c][MB], s);
      Msh[k][MB] = s / Msh[k][k];
    }
  }
  __syncwarp();
  double y = Msh[i][MB];
  if (lane < MB) g.x[i] = y;
  for (int b = 1; b < g.nb; ++b) {
    double S[MB], R[MB], w[1];
    load_row<MB>(g.data, b, i, S, R);
    w[0] = __ldg(g.f + (long)b * MB + i);
#pragma unroll
    for (int l = 0; l < MB; ++l) w[0] = fma(-S[l], gshfl<MB>(y, l), w[0]);
    lane_solve<MB, 1>(R, w, i);
    y = w[0];
    if (lane < MB) g.x[(long)b * MB + i] = y;
  }
}

}  // namespace psg
