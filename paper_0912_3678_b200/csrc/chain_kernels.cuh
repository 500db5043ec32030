// chain_kernels.cuh -- the partition method for the BVP layout of BABD
// (Kind::Babd with s = m, r = 0; BASELINE config 4):
//
//   block row 0       [ Ba                 ...   Bb(corner) ]   BC row
//   block row b >= 1  [ ... S_b  R_b ... ]                        x_b = R_b^-1 (f_b - S_b x_{b-1})
//
// i.e. a block lower-bidiagonal chain closed by the boundary condition.
// With separators sigma_0 = 0 < sigma_1 < ... < sigma_P = nb - 1 (the
// reference plan's separator blocks, src/partition.cpp:52-105), chunk j runs
// the chain over blocks sigma_j + 1 .. sigma_{j+1}:
//     x_{sigma_{j+1}} = Phi_j x_{sigma_j} + phi_j,
//     Phi_j = prod T_b, T_b = -R_b^-1 S_b      (factor: the body's F T G
//                                               blocks, src/localfact.cpp)
//     phi_j = the chain from 0 with f        (condense)
// The reduced system in x_sigma is again a BVP-layout BABD (R = I, S = -Phi,
// same Ba / Bb), solved by the same kernels recursively and finally by one
// warp (chain_direct_kernel, partial pivoting on the small BC system).  The
// final pass propagates x through every chunk and certifies the separator
// rows (componentwise backward error of the row S x_prev + R x_sep = f).
//
// MB lanes per chunk (lane i = row i of every block), 32 / MB chunks per
// warp; all shuffles are executed by the whole warp (chunk lengths differ by
// at most one step; shorter chunks idle through the last step).
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
template <int MB>
__global__ void __launch_bounds__(128) chain_factor_kernel(ChainLevelArgs g) {
  const int lane = threadIdx.x & 31, i = lane % MB;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) / MB;
  const bool live = j < g.P;
  const int b0 = live ? g.cut[j] + 1 : 1, b1 = live ? g.cut[j + 1] : 0;
  int len = b1 - b0 + 1, maxlen = len;
  for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
  double phi[MB];
#pragma unroll
  for (int c = 0; c < MB; ++c) phi[c] = i == c ? 1.0 : 0.0;
  for (int t = 0; t < maxlen; ++t) {
    const bool act = t < len;
    double S[MB], R[MB], w[MB];
    if (act) {
      load_row<MB>(g.data, b0 + t, i, S, R);
    } else {
#pragma unroll
      for (int c = 0; c < MB; ++c) {
        S[c] = 0.0;
        R[c] = i == c ? 1.0 : 0.0;
      }
    }
    // w = -S Phi (row i)
#pragma unroll
    for (int c = 0; c < MB; ++c) w[c] = 0.0;
#pragma unroll
    for (int l = 0; l < MB; ++l)
#pragma unroll
      for (int c = 0; c < MB; ++c) w[c] = fma(-S[l], gshfl<MB>(phi[c], l), w[c]);
    lane_solve<MB, MB>(R, w, i);
    if (act)
#pragma unroll
      for (int c = 0; c < MB; ++c) phi[c] = w[c];
  }
  if (live) {
    double* o = g.next_data + MB * MB + (long)j * 2 * MB * MB + (long)i * 2 * MB;
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      o[c] = -phi[c];
      o[MB + c] = i == c ? 1.0 : 0.0;
    }
    if (j == 0)
#pragma unroll
      for (int c = 0; c < MB; ++c) g.next_data[i * MB + c] = __ldg(g.data + i * MB + c);
  }
}

// condense: phi_j = the chain from zero with f; next_f[j+1] = phi_j, next_f[0] = f[0].
template <int MB>
__global__ void __launch_bounds__(128) chain_condense_kernel(ChainLevelArgs g) {
  const int lane = threadIdx.x & 31, i = lane % MB;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) / MB;
  const bool live = j < g.P;
  const int b0 = live ? g.cut[j] + 1 : 1, b1 = live ? g.cut[j + 1] : 0;
  int len = b1 - b0 + 1, maxlen = len;
  for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
  double y = 0.0;
  for (int t = 0; t < maxlen; ++t) {
    const bool act = t < len;
    double S[MB], R[MB], w[1];
    if (act) {
      load_row<MB>(g.data, b0 + t, i, S, R);
      w[0] = __ldg(g.f + (long)(b0 + t) * MB + i);
    } else {
#pragma unroll
      for (int c = 0; c < MB; ++c) {
        S[c] = 0.0;
        R[c] = i == c ? 1.0 : 0.0;
      }
      w[0] = 0.0;
    }
#pragma unroll
    for (int l = 0; l < MB; ++l) w[0] = fma(-S[l], gshfl<MB>(y, l), w[0]);
    lane_solve<MB, 1>(R, w, i);
    if (act) y = w[0];
  }
  if (live) {
    g.next_f[(long)(j + 1) * MB + i] = y;
    if (j == 0) g.next_f[i] = __ldg(g.f + i);
  }
}

__device__ __forceinline__ void cert_push(DevStatus* st, double num, double den) {
  double om = den > 0 ? num / den : num;
  if (!(om <= 1.0e308)) om = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) om = fmax(om, __shfl_xor_sync(0xffffffffu, om, o));
  if ((threadIdx.x & 31) == 0 && om > 0) status_cert(st, om);
}

// final: x through every chunk from its left separator value (next_x[j]);
// separator rows certified against next_x[j+1]; chunk 0 certifies the BC row.
// With corr_f, the separator residuals r are also condensed for one
// correction solve (A d = r, r living on the separator / BC rows only):
// corr_f[0] = r_BC, corr_f[j+1] = R_sep^-1 r_sep.  With accumulate, the pass
// is that correction: x += the homogeneous chain of d = next_x.
template <int MB>
__global__ void __launch_bounds__(128) chain_final_kernel(ChainLevelArgs g) {
  const int lane = threadIdx.x & 31, i = lane % MB;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) / MB;
  const bool live = j < g.P;
  const bool acc = g.accumulate != 0;
  const int b0 = live ? g.cut[j] + 1 : 1, b1 = live ? g.cut[j + 1] : 0;
  int len = b1 - b0 + 1, maxlen = len;
  for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
  // y: the chain (x, or d in the correction pass); yt: the value stored (x, or x_old + d)
  double y = live ? __ldg((acc ? g.corr_x : g.next_x) + (long)j * MB + i) : 0.0;
  double yt = (acc && live) ? __ldg(g.next_x + (long)j * MB + i) + y : y;
  if (live && j == 0) g.x[i] = yt;
  double num = 0.0, den = 0.0;
  bool finite = true;
  for (int t = 0; t < maxlen; ++t) {
    const bool act = t < len, last = t == len - 1;
    double S[MB], R[MB], w[2];
    double fv = 0.0, fs = 0.0;
    if (act) {
      load_row<MB>(g.data, b0 + t, i, S, R);
      if (!acc) fv = __ldg(g.f + (long)(b0 + t) * MB + i);
      if (acc && last) fs = __ldg(g.f + (long)(b0 + t) * MB + i);
    } else {
#pragma unroll
      for (int c = 0; c < MB; ++c) {
        S[c] = 0.0;
        R[c] = i == c ? 1.0 : 0.0;
      }
    }
    // separator row: residual of S x_prev + R x_sep = f with the reduced value
    // (acc: with the corrected values old x + d on both sides)
    const long os = (long)(b0 + t) * MB + i;
    const double xs = (act && last) ? __ldg((acc ? g.corr_x : g.next_x) + (long)(j + 1) * MB + i) : 0.0;
    const double xst = (acc && act && last) ? __ldg(g.next_x + (long)(j + 1) * MB + i) + xs : xs;
    double sg = 0.0, ab = 0.0;
    w[0] = fv;
#pragma unroll
    for (int l = 0; l < MB; ++l) {
      const double yl = gshfl<MB>(y, l), xl = gshfl<MB>(xst, l), ytl = gshfl<MB>(yt, l);
      const double p1 = S[l] * ytl, p2 = R[l] * xl;
      sg += p1 + p2;
      ab += fabs(p1) + fabs(p2);
      w[0] = fma(-S[l], yl, w[0]);
    }
    const double fr = acc ? fs : fv;
    w[1] = (act && last) ? fr - sg : 0.0;
    if (act && last) {
      const double om_num = fabs(fr - sg), om_den = fabs(fr) + ab;
      if (om_num * den > num * om_den || (den == 0.0 && om_num > 0)) {  // keep the max ratio
        num = om_num;
        den = om_den;
      }
    }
    lane_solve<MB, 2>(R, w, i);
    if (act) {
      y = last ? xs : w[0];
      yt = acc ? (last ? xst : g.x[os] + y) : y;
      finite &= isfinite(yt);
      g.x[os] = yt;
      if (last && g.corr_f) g.corr_f[(long)(j + 1) * MB + i] = w[1];
    }
  }
  if (!acc) {  // BC row (chunk 0): Ba x_0 + Bb x_{nb-1} = f_0; every group runs the shuffles
    const bool bc = live && j == 0;
    const double x0 = bc ? __ldg(g.next_x + i) : 0.0;
    const double xe = bc ? __ldg(g.next_x + (long)g.P * MB + i) : 0.0;
    double sg = 0.0, ab = 0.0;
#pragma unroll
    for (int l = 0; l < MB; ++l) {
      const double a0 = gshfl<MB>(x0, l), ae = gshfl<MB>(xe, l);
      if (bc) {
        const double p1 = __ldg(g.data + i * MB + l) * a0;
        const double p2 = __ldg(g.corner + i * MB + l) * ae;
        sg += p1 + p2;
        ab += fabs(p1) + fabs(p2);
      }
    }
    if (bc) {
      const double fv = __ldg(g.f + i);
      const double om_num = fabs(fv - sg), om_den = fabs(fv) + ab;
      if (om_num * den > num * om_den || (den == 0.0 && om_num > 0)) {
        num = om_num;
        den = om_den;
      }
      if (g.corr_f) g.corr_f[i] = fv - sg;
    }
  }
  if (!finite) num = __longlong_as_double(0x7ff0000000000000ll), den = 1.0;
  if (g.status) cert_push(g.status, num, den);
}

// componentwise backward error of the BC row Ba x_0 + Bb x_{nb-1} = f_0 (one warp)
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
