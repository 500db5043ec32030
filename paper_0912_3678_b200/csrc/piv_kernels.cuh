// piv_kernels.cuh -- the pivoting partition factorizations: Strategy::LuPivot
// and Strategy::Qr with adaptive reduced-system growth (reference
// src/localfact.cpp:517-607 lupivot_build / qr_build, dense_factor :674-760,
// condense :799-806, backsolve :850-875; src/parfact.cpp:72-127 kept blocks,
// :134-184 the reduced LU with partial pivoting), plus the no-pivot order of
// Strategy::Lu / Lud for the circulant-like kind, which has no other path.
//
// The reference materialises every body as a dense (k0+L+k1)^2 frame and
// records Lmat / Linv / Rmat.  Here one warp runs the SAME column sequence
// over a sliding window:
//
//   * rows live in 64 shared-memory slots: the active body rows (at most
//     es+1: rows enter at column x-es), the separator rows (top k0 loaded at
//     column 0, bottom k1 at column L-es-1) and the deferred rows;
//   * columns live in a 64-wide ring (body column c at ring c & 63; the pivot
//     row reaches c+es+er) plus up to 32 "spike" columns: left separator,
//     right separator, deferred columns;
//   * column c: pivot = max |W(row, c)| over the active rows, ties to the
//     lowest row (LuPivot), or a Householder reflector over the active rows
//     in ascending order (Qr); below tol * body_scale the lowest active row
//     and column c are deferred into the reduced system (an "extra");
//     otherwise column c is eliminated from every live row.
//
// Every frame entry receives its updates in the reference's order with the
// reference's roundings (no FMA, IEEE division and square root), so pivot
// choices, deferrals and the kept blocks (hence the reduced matrix T) are
// bit-identical to the reference.  The elimination steps are recorded
// (pivot slot, multipliers / reflector, pivot row) and replayed by the
// condense and backsolve kernels; the reduced system -- a band of half-width
// w = max kept dim - 1 (kept blocks [left sep | extras | right sep] are
// contiguous in position order) plus, for corner plans, a dense border of
// the last k columns -- is factored by the same engine in "dense LU" mode
// (tie-break by current row position, as the reference's row swaps do).
#pragma once

#include "gen_exact.cuh"

namespace psg {

constexpr int kPvRing = 64;   // ring columns (2 per lane)
constexpr int kPvSpk = 32;    // spike columns (1 per lane)
constexpr int kPvSlots = 64;  // live rows
constexpr int kPvRowW = kPvRing + kPvSpk + 1;  // odd pitch: column reads across rows are conflict-free

enum PivStrategy { kPvNoPivot = 0, kPvPartial = 1, kPvQr = 2 };

// Elimination records, one entry per step (body column / reduced column).
struct PivRec {
  int4* meta;            // {pivot slot or -1 (deferred), nt, na, deferred slot}
  unsigned char* tslot;  // NT per step: eliminated rows
  double* mu;            //   and their multipliers
  unsigned char* aslot;  // NA per step (Qr): reflector rows, ascending
  double* av;            //   reflector entries
  double* tau;           //   2 / v'v (0: no reflection)
  double* urow;          // URW per step: pivot row at columns c .. c+URW-1 (ring part)
  double* uspk;          // NS per step: pivot row at the spike columns
  int NT, NA, URW, NS;
};

struct PivArgs {
  SMView A;  // level 0 (canonical corner)
  const GPart* part;
  int p, k, es, er;
  int strategy;
  double tol;
  int cap;        // deferrals per body
  int KD;         // kept-block stride = 2k + cap
  double* kept;   // p x KD x KD, rows/cols [top sep | extras | bottom sep]
  int* ndef;      // p
  int* xpos;      // p x cap: body columns of the extras (ascending)
  // the reduced system
  double* rband;        // dim x (2w+1): column r-w+d of row r, columns below dim-kb
  double* rborder;      // dim x kb: columns dim-kb .. dim-1
  int dim, w, kb;
  PivRec rec;
  int* status;  // [0] exhausted body, [1] deferral capacity, [2] zero pivot (no-pivot order), [3] reduced singular
  // solve
  const double* f;    // rhs, global rows
  double* ghat;       // per step: the transformed rhs of the pivot row
  double* kr;         // p x KD kept rhs
  const double* rr;   // reduced rhs (reduced solve)
  double* xk;         // reduced solution
  const int* koff;    // per body: reduced offset of its kept block
  double* x;
};

struct PivSmem {
  double W[kPvSlots][kPvRowW];
  double mu[kPvSlots];
  int act[kPvSlots];  // active rows, ascending frame row (append order)
  int fst[kPvSlots];  // free-slot stack
  int tl[kPvSlots];   // targets of the current step
  int pos[kPvSlots];  // reduced mode: current row position (dense LU order)
  signed char st[kPvSlots];  // -1 free, 0 active, 3 separator, 4 deferred
  int sep[2 * kGenMaxK];
  int def[kPvSpk];
};

struct PivReplaySmem {
  double val[kPvSlots];
  double xr[kPvRing];
  double xs[kPvSpk];
  double av[kPvSlots];
  int fst[kPvSlots];
  int sep[2 * kGenMaxK];
  int def[kPvSpk];
};

__device__ __forceinline__ double pv_sub(double a, double m, double b) { return __dsub_rn(a, __dmul_rn(m, b)); }

// ---------------------------------------------------------------------------
// slot allocation: a stack, replayed identically by the condense kernels
// ---------------------------------------------------------------------------
__device__ __forceinline__ int pv_alloc(int* fst, int& top) {
  const int s = fst[top - 1];
  --top;
  return s;
}
__device__ __forceinline__ void pv_free(int* fst, int& top, int s) {
  __syncwarp();
  if (threadIdx.x == 0) fst[top] = s;
  ++top;
  __syncwarp();
}
__device__ __forceinline__ void pv_init_stack(int* fst, int& top) {
  for (int j = threadIdx.x; j < kPvSlots; j += 32) fst[j] = kPvSlots - 1 - j;
  top = kPvSlots;
  __syncwarp();
}

// Geometry of one elimination (a body, or the reduced system).
struct PvGeo {
  int L;       // columns stepped
  int k0, k1;  // separator rows / spike columns on each side
  int es, er;  // row reach below / above the diagonal
  int ring_end;  // columns >= ring_end live in the spike area (reduced border)
  int tb;      // step at which the bottom separator rows enter
};

// Which steps load which rows (the same schedule in factor and replay):
// step 0: top separator rows, rows 0..es; step t >= 1: row t+es; the bottom
// separator rows at step tb (after the body row of that step).
template <typename Fn>
__device__ __forceinline__ void pv_entering(const PvGeo& G, int t, Fn&& fn) {
  if (t == 0) {
    for (int u = 0; u < G.k0; ++u) fn(0, u);  // kind 0: top separator u
    for (int x = 0; x <= G.es && x < G.L; ++x) fn(1, x);
  } else if (t + G.es < G.L) {
    fn(1, t + G.es);
  }
  if (t == G.tb)
    for (int u = 0; u < G.k1; ++u) fn(2, u);
}

// Values of an entering row for the window [t, t + 64): ring slots lane and
// lane + 32 (v0, v1) and spike column lane (v2).  kind 0 / 1 / 2: top
// separator / body (or reduced) row / bottom separator.
template <int MODE>
__device__ __forceinline__ void pv_row_vals(const PivArgs& g, const GPart& P, const PvGeo& G, int kind, int idx,
                                            int t, double& v0, double& v1, double& v2) {
  const int lane = threadIdx.x;
  for (int h = 0; h < 2; ++h) {
    const int q = lane + 32 * h;
    const int c = t + ((q - t) & 63);  // column held by ring slot q in the window [t, t + 64)
    double v = 0.0;
    if (c < G.ring_end) {
      if (MODE == 1) {
        if (c >= idx - g.w && c <= idx + g.w) v = g.rband[(long)idx * (2 * g.w + 1) + (c - idx + g.w)];
      } else if (kind == 1) {
        if (c >= idx - G.es && c <= idx + G.er) v = sm_at(g.A, (long)P.b + idx, (long)P.b + c);
      } else {
        v = sm_at(g.A, kind == 0 ? (long)P.ls + idx : (long)P.rs + idx, (long)P.b + c);
      }
    }
    (h == 0 ? v0 : v1) = v;
  }
  double v = 0.0;
  if (MODE == 1) {
    if (lane < g.kb) v = g.rborder[(long)idx * g.kb + lane];
  } else if (kind == 1) {
    if (lane < G.k0) v = sm_at(g.A, (long)P.b + idx, (long)P.ls + lane);
    else if (lane < G.k0 + G.k1) v = sm_at(g.A, (long)P.b + idx, (long)P.rs + lane - G.k0);
  } else if (kind == 2) {  // right separator diagonal a_right; top x right-separator is zero in the frame
    if (lane >= G.k0 && lane < G.k0 + G.k1) v = sm_at(g.A, (long)P.rs + idx, (long)P.rs + lane - G.k0);
  }
  v2 = v;
}

// ---------------------------------------------------------------------------
// the factor engine
// ---------------------------------------------------------------------------
template <int MODE>  // 0: partition bodies (one warp each), 1: the reduced system (one warp)
__global__ void __launch_bounds__(32) piv_factor_kernel(PivArgs g) {
  extern __shared__ __align__(16) unsigned char pv_smem_raw[];
  PivSmem& S = *reinterpret_cast<PivSmem*>(pv_smem_raw);
  const int lane = threadIdx.x;
  const int body = blockIdx.x;
  GPart P{0, 0, -1, -1};
  PvGeo G;
  if (MODE == 0) {
    P = g.part[body];
    G.L = P.L;
    G.k0 = P.ls >= 0 ? g.k : 0;
    G.k1 = P.rs >= 0 ? g.k : 0;
    G.es = min(g.es, P.L - 1);
    G.er = min(g.er, P.L - 1);
    G.ring_end = P.L;
    G.tb = max(0, P.L - G.es - 1);
  } else {
    G.L = g.dim;
    G.k0 = G.k1 = 0;
    G.es = G.er = g.w;
    G.ring_end = g.dim - g.kb;
    G.tb = -1;
  }
  const long rbase = MODE == 0 ? (long)P.b : 0;  // record index of step 0
  const int strategy = MODE == 0 ? g.strategy : kPvPartial;

  // body_scale (src/localfact.cpp:63-72): max over body rows of sum |env|
  double tolsc = 0.0;
  if (MODE == 0 && strategy != kPvNoPivot) {
    double sc = 1e-300;
    for (int x = lane; x < G.L; x += 32) {
      double s = 0.0;
      for (int d = -G.es; d <= G.er; ++d) {
        const int c = x + d;
        const double v = (c >= 0 && c < G.L) ? sm_at(g.A, (long)P.b + x, (long)P.b + c) : 0.0;
        s = __dadd_rn(s, fabs(v));
      }
      sc = fmax(sc, s);
    }
    for (int o = 16; o > 0; o >>= 1) sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, o));
    tolsc = __dmul_rn(g.tol, sc);
  }

  int top;
  pv_init_stack(S.fst, top);
  for (int j = lane; j < kPvSlots; j += 32) S.st[j] = -1;
  for (int j = 0; j < kPvSlots; ++j)
    for (int c = lane; c < kPvRowW; c += 32) S.W[j][c] = 0.0;
  __syncwarp();
  int nact = 0, ndef = 0;
  bool failed = false;

  // entering body / reduced rows of steps t + 1 and t + 2, prefetched into registers
  double pa0 = 0.0, pa1 = 0.0, pa2 = 0.0, pb0 = 0.0, pb1 = 0.0, pb2 = 0.0;
  if (1 + G.es < G.L) pv_row_vals<MODE>(g, P, G, 1, 1 + G.es, 1, pa0, pa1, pa2);
  if (2 + G.es < G.L) pv_row_vals<MODE>(g, P, G, 1, 2 + G.es, 2, pb0, pb1, pb2);
  for (int t = 0; t < G.L && !failed; ++t) {
    // ---- rows entering at this step (the order pv_entering replays)
    pv_entering(G, t, [&](int kind, int idx) {
      const int sl = pv_alloc(S.fst, top);
      double v0, v1, v2;
      if (kind == 1 && t >= 1) {
        v0 = pa0;
        v1 = pa1;
        v2 = pa2;
      } else {
        pv_row_vals<MODE>(g, P, G, kind, idx, t, v0, v1, v2);
      }
      S.W[sl][lane] = v0;
      S.W[sl][lane + 32] = v1;
      S.W[sl][kPvRing + lane] = v2;
      if (lane == 0) {
        if (kind == 1) {
          S.st[sl] = 0;
          S.act[nact] = sl;
          S.pos[sl] = idx;
        } else {
          S.st[sl] = 3;
          S.sep[kind == 0 ? idx : G.k0 + idx] = sl;
        }
      }
      if (kind == 1) ++nact;
      __syncwarp();
    });
    if (t >= 1) {  // pa held step t's row: shift, fetch step t + 2's
      pa0 = pb0;
      pa1 = pb1;
      pa2 = pb2;
      if (t + 2 + G.es < G.L) pv_row_vals<MODE>(g, P, G, 1, t + 2 + G.es, t + 2, pb0, pb1, pb2);
    }

    const int c = t;
    const int pc = c < G.ring_end ? (c & 63) : kPvRing + (c - G.ring_end);
    const long ri = rbase + t;

    // ---- pivot choice (or the reflector norm)
    int piv = -1;
    bool defer = false;
    double nrm = 0.0;
    if (strategy == kPvQr) {
      double n2 = 0.0;
      for (int u = 0; u < nact; ++u) {
        const double xv = S.W[S.act[u]][pc];
        n2 = __dadd_rn(n2, __dmul_rn(xv, xv));
      }
      nrm = __dsqrt_rn(n2);
      defer = nrm < tolsc;
    } else if (strategy == kPvNoPivot) {
      piv = S.act[0];
      if (S.W[piv][pc] == 0.0) {
        if (lane == 0) atomicMin(g.status + 2, body);
        failed = true;
        break;
      }
    } else {
      double bv = -1.0;
      int bkey = INT_MAX, bsl = -1;
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (j < nact) {
          const int sl = S.act[j];
          double v = fabs(S.W[sl][pc]);
          if (!(v == v)) v = -1.0;  // NaN never wins the reference's strict '>'
          const int key = MODE == 0 ? j : S.pos[sl];
          if (v > bv || (v == bv && key < bkey)) {
            bv = v;
            bkey = key;
            bsl = sl;
          }
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int ok = __shfl_xor_sync(0xffffffffu, bkey, o);
        const int os = __shfl_xor_sync(0xffffffffu, bsl, o);
        if (ov > bv || (ov == bv && ok < bkey)) {
          bv = ov;
          bkey = ok;
          bsl = os;
        }
      }
      if (MODE == 1) {
        if (bv == 0.0 || bsl < 0) {
          if (lane == 0) atomicMin(g.status + 3, 0);
          failed = true;
          break;
        }
      } else {
        defer = bv < tolsc;
      }
      piv = bsl;
    }

    if (defer) {  // ---- the lowest active row and column c join the reduced system
      const int rho = S.act[0];
      if (ndef >= g.cap || G.k0 + G.k1 + ndef >= kPvSpk) {
        if (lane == 0) atomicMin(g.status + 1, body);
        failed = true;
        break;
      }
      const int sc = kPvRing + G.k0 + G.k1 + ndef;
      for (int h = 0; h < 2; ++h) {
        const int sl = lane + 32 * h;
        if (S.st[sl] >= 0) {
          S.W[sl][sc] = S.W[sl][pc];
          S.W[sl][pc] = 0.0;
        }
      }
      __syncwarp();
      // drop act[0]
      int nv = 0;
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (j + 1 < nact) nv = S.act[j + 1];
        __syncwarp();
        if (j + 1 < nact) S.act[j] = nv;
        __syncwarp();
      }
      --nact;
      if (lane == 0) {
        S.st[rho] = 4;
        S.def[ndef] = rho;
        g.xpos[(long)body * g.cap + ndef] = c;
        g.rec.meta[ri] = make_int4(-1, 0, 0, rho);
      }
      ++ndef;
      __syncwarp();
      continue;
    }

    int na = 0;
    double tau = 0.0;
    if (strategy == kPvQr) {  // ---- Householder reflector over the active rows (src/localfact.cpp:575-597)
      na = nact;
      const double x0 = S.W[S.act[0]][pc];
      const double alpha = x0 >= 0 ? -nrm : nrm;
      double vtv = 0.0;
      for (int u = 0; u < na; ++u) {
        double vu = S.W[S.act[u]][pc];
        if (u == 0) vu = __dsub_rn(vu, alpha);
        vtv = __dadd_rn(vtv, __dmul_rn(vu, vu));
      }
      __syncwarp();
      for (int h = 0; h < 2; ++h) {
        const int u = lane + 32 * h;
        if (u < na) {
          double vu = S.W[S.act[u]][pc];
          if (u == 0) vu = __dsub_rn(vu, alpha);
          S.mu[u] = vu;
        }
      }
      __syncwarp();
      if (vtv > 0.0) {
        tau = __ddiv_rn(2.0, vtv);
        for (int h = 0; h < 3; ++h) {
          const int col = h < 2 ? lane + 32 * h : kPvRing + lane;
          double s = 0.0;
          for (int u = 0; u < na; ++u) s = __dadd_rn(s, __dmul_rn(S.mu[u], S.W[S.act[u]][col]));
          s = __dmul_rn(s, tau);
          for (int u = 0; u < na; ++u) S.W[S.act[u]][col] = pv_sub(S.W[S.act[u]][col], s, S.mu[u]);
        }
        __syncwarp();
      }
      if (lane == (pc & 31)) {  // the lane owning column pc writes the reflected column
        for (int u = 0; u < na; ++u) S.W[S.act[u]][pc] = u == 0 ? alpha : 0.0;
      }
      __syncwarp();
      if (lane < na) {
        g.rec.aslot[ri * g.rec.NA + lane] = (unsigned char)S.act[lane];
        g.rec.av[ri * g.rec.NA + lane] = S.mu[lane];
      }
      if (lane == 0) g.rec.tau[ri] = tau;
      piv = S.act[0];
      __syncwarp();
    }

    // ---- retire the pivot row; reduced mode swaps it into position c
    {
      int idx = -1;
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        const unsigned b = __ballot_sync(0xffffffffu, j < nact && S.act[j] == piv);
        if (b && idx < 0) idx = 32 * h + __ffs(b) - 1;
      }
      if (MODE == 1) {
        const int ppos = S.pos[piv];
        __syncwarp();
        for (int h = 0; h < 2; ++h) {
          const int j = lane + 32 * h;
          if (j < nact && S.pos[S.act[j]] == c && S.act[j] != piv) S.pos[S.act[j]] = ppos;
        }
        __syncwarp();
        if (lane == 0) S.pos[piv] = c;
      }
      int nv = 0;
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (j >= idx && j + 1 < nact) nv = S.act[j + 1];
        __syncwarp();
        if (j >= idx && j + 1 < nact) S.act[j] = nv;
        __syncwarp();
      }
      --nact;
      if (lane == 0) S.st[piv] = 1;
      __syncwarp();
    }

    // ---- eliminate column c from the live rows (Qr: separator / deferred rows only)
    int nt = 0;
    {
      const double pvv = S.W[piv][pc];
      for (int h = 0; h < 2; ++h) {
        const int sl = lane + 32 * h;
        const int stv = S.st[sl];
        const bool elig = strategy == kPvQr ? (stv == 3 || stv == 4) : (stv == 0 || stv == 3 || stv == 4);
        const bool tg = elig && S.W[sl][pc] != 0.0;
        const unsigned b = __ballot_sync(0xffffffffu, tg);
        if (tg) {
          const int at = nt + __popc(b & ((1u << lane) - 1u));
          S.tl[at] = sl;
          S.mu[sl] = __ddiv_rn(S.W[sl][pc], pvv);
        }
        nt += __popc(b);
      }
      __syncwarp();
      const double p0 = S.W[piv][lane], p1 = S.W[piv][lane + 32], p2 = S.W[piv][kPvRing + lane];
      for (int i = 0; i < nt; ++i) {
        const int sl = S.tl[i];
        const double m = S.mu[sl];
        S.W[sl][lane] = pv_sub(S.W[sl][lane], m, p0);
        S.W[sl][lane + 32] = pv_sub(S.W[sl][lane + 32], m, p1);
        S.W[sl][kPvRing + lane] = pv_sub(S.W[sl][kPvRing + lane], m, p2);
      }
      __syncwarp();
      for (int i = lane; i < nt; i += 32) S.W[S.tl[i]][pc] = 0.0;
      __syncwarp();
    }

    // ---- record the step, free the pivot slot
    for (int i = lane; i < nt; i += 32) {
      g.rec.tslot[ri * g.rec.NT + i] = (unsigned char)S.tl[i];
      g.rec.mu[ri * g.rec.NT + i] = S.mu[S.tl[i]];
    }
    for (int j = lane; j < g.rec.URW; j += 32) {
      const int cc = c + j;
      g.rec.urow[ri * g.rec.URW + j] = cc < G.ring_end ? S.W[piv][cc & 63] : 0.0;
    }
    if (lane < g.rec.NS) g.rec.uspk[ri * g.rec.NS + lane] = S.W[piv][kPvRing + lane];
    if (lane == 0) g.rec.meta[ri] = make_int4(piv, nt, na, -1);
    __syncwarp();
    S.W[piv][lane] = 0.0;
    S.W[piv][lane + 32] = 0.0;
    S.W[piv][kPvRing + lane] = 0.0;
    if (lane == 0) S.st[piv] = -1;
    pv_free(S.fst, top, piv);
  }
  if (MODE == 1 || failed) return;

  // ---- the kept block: rows / cols [top separator | deferred (in order) | bottom separator]
  if (ndef == G.L && lane == 0) atomicMin(g.status + 0, body);
  if (lane == 0) g.ndef[body] = ndef;
  const int kd = G.k0 + ndef + G.k1;
  for (int a = 0; a < kd; ++a) {
    const int sl = a < G.k0 ? S.sep[a] : (a < G.k0 + ndef ? S.def[a - G.k0] : S.sep[G.k0 + (a - G.k0 - ndef)]);
    if (lane < kd) {
      const int b = lane;
      const int sc = b < G.k0 ? b : (b < G.k0 + ndef ? G.k0 + G.k1 + (b - G.k0) : G.k0 + (b - G.k0 - ndef));
      g.kept[((long)body * g.KD + a) * g.KD + b] = S.W[sl][kPvRing + sc];
    }
  }
}

// One step's records, loaded a step ahead (they do not depend on the data).
struct PvStepRec {
  int4 mt;
  int s0, s1;        // target slots of entries lane, lane + 32
  double m0, m1;     // their multipliers
  int a0;            // Qr: reflector slot / entry of lane
  double av0, tau;
};

__device__ __forceinline__ PvStepRec pv_load_rec(const PivRec& R, long ri) {
  const int lane = threadIdx.x;
  PvStepRec r;
  r.mt = R.meta[ri];
  r.s0 = lane < R.NT ? R.tslot[ri * R.NT + lane] : 0;
  r.m0 = lane < R.NT ? R.mu[ri * R.NT + lane] : 0.0;
  r.s1 = lane + 32 < R.NT ? R.tslot[ri * R.NT + lane + 32] : 0;
  r.m1 = lane + 32 < R.NT ? R.mu[ri * R.NT + lane + 32] : 0.0;
  r.a0 = lane < R.NA ? R.aslot[ri * R.NA + lane] : 0;
  r.av0 = lane < R.NA ? R.av[ri * R.NA + lane] : 0.0;
  r.tau = R.tau[ri];
  return r;
}

// Apply one recorded elimination step to the slot values (condense replay).
__device__ __forceinline__ void pv_apply_rec(double* val, const PvStepRec& r, double* ghat_out, double* av) {
  const int lane = threadIdx.x;
  if (r.mt.z > 0) {  // Qr reflector: s = tau * sum_u v_u val[rows_u]
    if (lane < r.mt.z) av[lane] = r.av0;
    __syncwarp();
    double part = lane < r.mt.z ? __dmul_rn(r.av0, val[r.a0]) : 0.0;
    double sum = 0.0;
    for (int u = 0; u < r.mt.z; ++u) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, part, u));
    sum = __dmul_rn(sum, r.tau);
    __syncwarp();
    if (lane < r.mt.z) val[r.a0] = pv_sub(val[r.a0], sum, r.av0);
    __syncwarp();
  }
  const double pv = val[r.mt.x];
  if (lane == 0 && ghat_out) *ghat_out = pv;
  if (lane < r.mt.y) val[r.s0] = pv_sub(val[r.s0], r.m0, pv);
  if (lane + 32 < r.mt.y) val[r.s1] = pv_sub(val[r.s1], r.m1, pv);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// condense replay (phase 1) for the bodies: ghat per step, kept rhs per body
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32) piv_condense_kernel(PivArgs g) {
  __shared__ PivReplaySmem S;
  const int lane = threadIdx.x, body = blockIdx.x;
  const GPart P = g.part[body];
  PvGeo G;
  G.L = P.L;
  G.k0 = P.ls >= 0 ? g.k : 0;
  G.k1 = P.rs >= 0 ? g.k : 0;
  G.es = min(g.es, P.L - 1);
  G.er = min(g.er, P.L - 1);
  G.ring_end = P.L;
  G.tb = max(0, P.L - G.es - 1);
  int top;
  pv_init_stack(S.fst, top);
  int nd = 0;
  PvStepRec cur = pv_load_rec(g.rec, P.b), nxt = cur;
  if (G.L > 1) nxt = pv_load_rec(g.rec, (long)P.b + 1);
  double fin = (1 + G.es < G.L) ? g.f[(long)P.b + 1 + G.es] : 0.0;  // entering rhs of step t + 1
  for (int t = 0; t < G.L; ++t) {
    pv_entering(G, t, [&](int kind, int idx) {
      const int sl = pv_alloc(S.fst, top);
      if (lane == 0) {
        S.val[sl] = kind == 1 ? (t >= 1 ? fin : g.f[(long)P.b + idx]) : 0.0;
        if (kind != 1) S.sep[kind == 0 ? idx : G.k0 + idx] = sl;
      }
      __syncwarp();
    });
    fin = (t + 1 + G.es < G.L) ? g.f[(long)P.b + t + 1 + G.es] : 0.0;  // step t + 1's entering rhs
    const PvStepRec r = cur;
    cur = nxt;
    if (t + 2 < G.L) nxt = pv_load_rec(g.rec, (long)P.b + t + 2);
    if (r.mt.x < 0) {
      if (lane == 0) S.def[nd] = r.mt.w;
      ++nd;
      __syncwarp();
      continue;
    }
    pv_apply_rec(S.val, r, g.ghat + (long)P.b + t, S.av);
    pv_free(S.fst, top, r.mt.x);
  }
  const int kd = G.k0 + nd + G.k1;
  for (int a = lane; a < kd; a += 32) {
    const int sl = a < G.k0 ? S.sep[a] : (a < G.k0 + nd ? S.def[a - G.k0] : S.sep[G.k0 + (a - G.k0 - nd)]);
    g.kr[(long)body * g.KD + a] = S.val[sl];
  }
}

// Back-substitution records of one step, loaded a step ahead.
struct PvBackRec {
  int4 mt;
  double u0, u1, us, diag, gh;
};

__device__ __forceinline__ PvBackRec pv_load_back(const PivRec& R, const double* ghat, long ri) {
  const int lane = threadIdx.x;
  PvBackRec b;
  b.mt = R.meta[ri];
  b.u0 = lane + 1 < R.URW ? R.urow[ri * R.URW + lane + 1] : 0.0;
  b.u1 = lane + 33 < R.URW ? R.urow[ri * R.URW + lane + 33] : 0.0;
  b.us = lane < R.NS ? R.uspk[ri * R.NS + lane] : 0.0;
  b.diag = R.urow[ri * R.URW];
  b.gh = ghat[ri];
  return b;
}

// ---------------------------------------------------------------------------
// backsolve replay (phase 3) for the bodies, plus the separators they own
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32) piv_backsolve_kernel(PivArgs g) {
  __shared__ PivReplaySmem S;
  const int lane = threadIdx.x, body = blockIdx.x;
  const GPart P = g.part[body];
  const int L = P.L, k0 = P.ls >= 0 ? g.k : 0, k1 = P.rs >= 0 ? g.k : 0;
  const int nd = g.ndef[body];
  const int ko = g.koff[body];
  // spike values: left separator, right separator, extras
  double xsv = 0.0;
  if (lane < k0) xsv = g.xk[ko + lane];
  else if (lane < k0 + k1) xsv = g.xk[ko + k0 + nd + (lane - k0)];
  else if (lane < k0 + k1 + nd) xsv = g.xk[ko + k0 + (lane - k0 - k1)];
  S.xs[lane] = xsv;
  S.xr[lane] = 0.0;
  S.xr[lane + 32] = 0.0;
  __syncwarp();
  int d = nd - 1;
  PvBackRec cur = pv_load_back(g.rec, g.ghat, (long)P.b + L - 1), nxt = cur;
  if (L > 1) nxt = pv_load_back(g.rec, g.ghat, (long)P.b + L - 2);
  for (int t = L - 1; t >= 0; --t) {
    const PvBackRec r = cur;
    cur = nxt;
    if (t >= 2) nxt = pv_load_back(g.rec, g.ghat, (long)P.b + t - 2);
    double xv;
    if (r.mt.x < 0) {
      xv = g.xk[ko + k0 + d];
      --d;
    } else {
      double acc = 0.0;
      if (t + lane + 1 < L) acc = __fma_rn(r.u0, S.xr[(t + lane + 1) & 63], acc);
      if (t + lane + 33 < L) acc = __fma_rn(r.u1, S.xr[(t + lane + 33) & 63], acc);
      acc = __fma_rn(r.us, S.xs[lane], acc);
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      xv = (r.gh - acc) / r.diag;
    }
    __syncwarp();
    if (lane == 0) {
      S.xr[t & 63] = xv;
      g.x[(long)P.b + t] = xv;
    }
    __syncwarp();
  }
  // separators: each written by the body on its left (corner plans: body 0 also writes separator 0)
  if (lane < k1) g.x[(long)P.rs + lane] = g.xk[ko + k0 + nd + lane];
  if (body == 0 && lane < k0) g.x[(long)P.ls + lane] = g.xk[ko + lane];
}

// ---------------------------------------------------------------------------
// the reduced system: assembly (two passes keep the reference's summation
// order: central corner terms, then kept blocks in partition order)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pv_rput(const PivArgs& g, int row, int col, double v, bool add) {
  double* dst = col >= g.dim - g.kb ? g.rborder + (long)row * g.kb + (col - (g.dim - g.kb))
                                    : g.rband + (long)row * (2 * g.w + 1) + (col - row + g.w);
  *dst = add ? __dadd_rn(*dst, v) : v;
}

template <int PASS>  // 0: rows below the top separator (exclusive), + the central corner terms; 1: top rows (add)
__global__ void __launch_bounds__(32) piv_assemble_kernel(PivArgs g) {
  const int lane = threadIdx.x, body = blockIdx.x;
  const GPart P = g.part[body];
  const int k0 = P.ls >= 0 ? g.k : 0, k1 = P.rs >= 0 ? g.k : 0;
  const int nd = g.ndef[body], kd = k0 + nd + k1, ko = g.koff[body];
  for (int a = PASS == 0 ? k0 : 0; a < (PASS == 0 ? kd : k0); ++a)
    for (int b = lane; b < kd; b += 32) pv_rput(g, ko + a, ko + b, g.kept[((long)body * g.KD + a) * g.KD + b], PASS == 1);
  if (PASS == 0 && body == 0 && P.ls >= 0) {
    // corner plans (src/parfact.cpp:94-104): separator 0's own diagonal and the corner slice
    const int sp = g.part[g.p - 1].rs, o0 = ko, op = g.dim - g.k;
    for (int t = 0; t < g.k; ++t)
      for (int u = lane; u < g.k; u += 32) {
        pv_rput(g, o0 + t, o0 + u, sm_at(g.A, (long)P.ls + t, (long)P.ls + u), false);
        pv_rput(g, o0 + t, op + u, sm_at(g.A, (long)P.ls + t, (long)sp + u), false);
      }
  }
}

// reduced rhs (src/parfact.cpp:205-214): separators start from f, then every
// partition adds its kept rhs in partition order
__global__ void piv_rrhs_kernel(PivArgs g, double* rr) {
  const int lane = threadIdx.x, body = blockIdx.x;
  const GPart P = g.part[body];
  const int k0 = P.ls >= 0 ? g.k : 0, k1 = P.rs >= 0 ? g.k : 0;
  const int nd = g.ndef[body], ko = g.koff[body];
  const double* kr = g.kr + (long)body * g.KD;
  for (int a = lane; a < nd; a += 32) rr[ko + k0 + a] = kr[k0 + a];
  if (lane < k1) {
    double v = __dadd_rn(g.f[(long)P.rs + lane], kr[k0 + nd + lane]);
    if (body + 1 < g.p) v = __dadd_rn(v, g.kr[(long)(body + 1) * g.KD + lane]);  // next body's top rows
    rr[ko + k0 + nd + lane] = v;
  }
  if (body == 0 && lane < k0) rr[ko + lane] = __dadd_rn(g.f[(long)P.ls + lane], kr[lane]);
}

// The reduced solve (one warp): replay the reduced LU on rr, back-substitute.
__global__ void __launch_bounds__(32) piv_reduced_solve_kernel(PivArgs g) {
  __shared__ PivReplaySmem S;
  const int lane = threadIdx.x;
  PvGeo G;
  G.L = g.dim;
  G.k0 = G.k1 = 0;
  G.es = G.er = g.w;
  G.ring_end = g.dim - g.kb;
  G.tb = -1;
  int top;
  pv_init_stack(S.fst, top);
  PvStepRec cur = pv_load_rec(g.rec, 0), nxt = cur;
  if (G.L > 1) nxt = pv_load_rec(g.rec, 1);
  double fin = (1 + G.es < G.L) ? g.rr[1 + G.es] : 0.0;
  for (int t = 0; t < G.L; ++t) {
    pv_entering(G, t, [&](int, int idx) {
      const int sl = pv_alloc(S.fst, top);
      if (lane == 0) S.val[sl] = t >= 1 ? fin : g.rr[idx];
      __syncwarp();
    });
    fin = (t + 1 + G.es < G.L) ? g.rr[t + 1 + G.es] : 0.0;  // step t + 1's entering rhs
    const PvStepRec r = cur;
    cur = nxt;
    if (t + 2 < G.L) nxt = pv_load_rec(g.rec, t + 2);
    pv_apply_rec(S.val, r, g.ghat + t, S.av);
    pv_free(S.fst, top, r.mt.x);
  }
  S.xr[lane] = 0.0;
  S.xr[lane + 32] = 0.0;
  S.xs[lane] = 0.0;
  __syncwarp();
  __threadfence_block();
  PvBackRec bc = pv_load_back(g.rec, g.ghat, G.L - 1), bn = bc;
  if (G.L > 1) bn = pv_load_back(g.rec, g.ghat, G.L - 2);
  for (int t = G.L - 1; t >= 0; --t) {
    const PvBackRec r = bc;
    bc = bn;
    if (t >= 2) bn = pv_load_back(g.rec, g.ghat, t - 2);
    const bool spike = t >= G.ring_end;
    const int sown = spike ? t - G.ring_end : -1;
    double acc = 0.0;
    if (!spike) {
      if (t + lane + 1 < G.ring_end) acc = __fma_rn(r.u0, S.xr[(t + lane + 1) & 63], acc);
      if (t + lane + 33 < G.ring_end) acc = __fma_rn(r.u1, S.xr[(t + lane + 33) & 63], acc);
    }
    if (lane < g.kb && lane != sown) acc = __fma_rn(r.us, S.xs[lane], acc);
    const double dgs = __shfl_sync(0xffffffffu, r.us, sown < 0 ? 0 : sown);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const double xv = (r.gh - acc) / (spike ? dgs : r.diag);
    __syncwarp();
    if (lane == 0) {
      if (spike) S.xs[sown] = xv;
      else S.xr[t & 63] = xv;
      g.xk[t] = xv;
    }
    __syncwarp();
  }
}

// circulant-like rows rotated down by r (src/partition.cpp:175-202): out[i] = in[(i - r) mod n]
__global__ void piv_rotate_kernel(long n, long rows, int r, const double* __restrict__ in, double* __restrict__ out) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < n * rows; t += stride) {
    const long q = t / n, i = t - q * n;
    long src = i - r;
    if (src < 0) src += n;
    out[t] = in[q * n + src];
  }
}

}  // namespace psg
