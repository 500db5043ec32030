// host_localfact.cpp -- LocalFactorization and the factor_* entry points of
// the C++ API (reference proj/include/parsol/localfact.hpp:24-125) over the
// C ABI psg_local_* (csrc/psg_local.cu).
//
// factor_*: the partition block goes to the device, one CTA factors it, and
// every field of the reference's LocalFactorization comes back as a host view
// (bit-identical values).  The member operations run on the device against
// the same factorization.  The dense_* materializations are assembled here on
// the host from those views: they are the reference's test oracles (its
// header: "Only tests build these; the solver never forms F, T, G").
#include <algorithm>
#include <string>

#include "parsol/localfact.hpp"
#include "psg.h"

namespace parsol {

namespace {

void check(int rc, const char* err) {
  if (rc) fail(Errc(rc - 1), err);
}

DenseMatrix read_mat(const psg_local* h, int field, int rows, int cols) {
  DenseMatrix M(rows, cols);
  if (rows == 0 || cols == 0) return M;
  char err[256];
  check(psg_local_read(h, field, M.a.data(), M.a.size(), err, sizeof err), err);
  return M;
}

std::vector<int> read_ints(const psg_local* h, int field, int count) {
  std::vector<int> v(std::max(count, 0));
  if (count <= 0) return v;
  char err[256];
  check(psg_local_read(h, field, v.data(), v.size(), err, sizeof err), err);
  return v;
}

// g x g block q of a packed array of blocks
DenseMatrix block_at(const std::vector<double>& packed, int q, int g) {
  DenseMatrix B(g, g);
  std::copy_n(packed.begin() + std::size_t(q) * g * g, std::size_t(g) * g, B.a.begin());
  return B;
}

LocalFactorization run_factor(const PartitionBlock& M, Strategy s, double tol) {
  psg_block b{};
  b.kind = int(M.kind);
  b.m = M.m;
  b.s = M.s;
  b.r = M.r;
  b.L = M.L;
  b.k0 = M.k0;
  b.k1 = M.k1;
  b.env_s = M.env_s;
  b.env_r = M.env_r;
  b.env = M.env.data();
  auto ptr = [](const DenseMatrix& D) { return D.a.empty() ? nullptr : D.a.data(); };
  b.b0 = ptr(M.b0);
  b.c0 = ptr(M.c0);
  b.b1 = ptr(M.b1);
  b.c1 = ptr(M.c1);
  b.a_right = ptr(M.a_right);
  if (std::size_t(M.L) * (M.env_s + 1 + M.env_r) != M.env.size())
    fail(Errc::DimensionMismatch, "partition block envelope size");
  psg_local* raw = nullptr;
  char err[512];
  check(psg_local_factor(&b, int(s), tol, nullptr, &raw, err, sizeof err), err);
  std::shared_ptr<psg_local> dev(raw, psg_local_release);
  psg_local_info in{};
  psg_local_query(raw, &in);

  LocalFactorization lf;
  lf.strategy = s;
  lf.L = M.L;
  lf.k0 = M.k0;
  lf.k1 = M.k1;
  lf.device = dev;
  const int L = M.L, k0 = M.k0, k1 = M.k1;
  if (in.core == 1 || in.core == 3) {
    lf.z = read_mat(raw, PSG_LF_Z, L, k0);
    lf.w = read_mat(raw, PSG_LF_W, L, k0);
    lf.y = read_mat(raw, PSG_LF_Y, L, k1);
    lf.v = read_mat(raw, PSG_LF_V, L, k1);
  }
  lf.alpha1 = read_mat(raw, PSG_LF_ALPHA1, k0, k0);
  lf.alpha2 = read_mat(raw, PSG_LF_ALPHA2, k1, k1);
  lf.beta = read_mat(raw, PSG_LF_BETA, k1, k0);
  lf.gamma = read_mat(raw, PSG_LF_GAMMA, k0, k1);
  const int nx = in.n_extras;
  if (in.core == 3) {
    const std::vector<int> pos = read_ints(raw, PSG_LF_EXTRA_POS, nx);
    std::vector<double> alpha(nx);
    if (nx) check(psg_local_read(raw, PSG_LF_EXTRA_ALPHA, alpha.data(), alpha.size(), err, sizeof err), err);
    for (int u = 0; u < nx; ++u) lf.extras.push_back({pos[u], alpha[u]});
  }
  const int kd = k0 + nx + k1;
  lf.kept = read_mat(raw, PSG_LF_KEPT, kd, kd);

  if (in.core == 1) {
    LocalFactorization::BandedCore c;
    c.L = L;
    c.es = M.env_s;
    c.er = M.env_r;
    c.unit_mid = s == Strategy::Lud;
    c.fac.resize(M.env.size());
    check(psg_local_read(raw, PSG_LF_FAC, c.fac.data(), c.fac.size(), err, sizeof err), err);
    if (c.unit_mid) {
      c.dvec.resize(L);
      check(psg_local_read(raw, PSG_LF_DVEC, c.dvec.data(), c.dvec.size(), err, sizeof err), err);
    }
    lf.core = std::move(c);
  } else if (in.core == 2) {
    LocalFactorization::CyclicCore c;
    c.g = in.g;
    c.nb = L / in.g;
    const int g = c.g, gg = g * g, ne = in.n_elims, rg = in.n_rem * g;
    lf.cr_levels = in.cr_levels;
    const std::vector<int> idx = read_ints(raw, PSG_LF_CR_ELIM_IDX, 3 * ne);
    std::vector<double> mats(std::size_t(ne) * 5 * gg);
    if (ne) check(psg_local_read(raw, PSG_LF_CR_ELIM_MAT, mats.data(), mats.size(), err, sizeof err), err);
    for (int q = 0; q < ne; ++q) {
      LocalFactorization::CyclicCore::Elim e;
      e.j = idx[3 * q];
      e.lnb = idx[3 * q + 1];
      e.rnb = idx[3 * q + 2];
      e.ml = block_at(mats, 5 * q, g);
      e.mr = block_at(mats, 5 * q + 1, g);
      e.a = block_at(mats, 5 * q + 2, g);
      e.c = block_at(mats, 5 * q + 3, g);
      e.dinv = block_at(mats, 5 * q + 4, g);
      c.elims.push_back(std::move(e));
    }
    for (int u = 0; u < in.n_rem; ++u) c.rem.push_back(in.rem[u]);
    c.d2 = read_mat(raw, PSG_LF_CR_D2, rg, rg);
    c.d2inv = read_mat(raw, PSG_LF_CR_D2INV, rg, rg);
    c.cmat = read_mat(raw, PSG_LF_CR_CMAT, rg, k0 + k1);
    c.rmat_d2inv = read_mat(raw, PSG_LF_CR_RMAT_D2INV, k0 + k1, rg);
    lf.core = std::move(c);
  } else {
    LocalFactorization::DenseCore c;
    c.dim = in.dim;
    c.Wmid = read_mat(raw, PSG_LF_WMID, in.dim, in.dim);
    c.Lmat = read_mat(raw, PSG_LF_LMAT, in.dim, in.dim);
    c.Linv = read_mat(raw, PSG_LF_LINV, in.dim, in.dim);
    const std::vector<int> ao = read_ints(raw, PSG_LF_A_ORDER, 2 * in.n_a_order);
    for (int q = 0; q < in.n_a_order; ++q) {
      c.a_order.emplace_back(ao[2 * q], ao[2 * q + 1]);
      lf.row_perm.push_back(ao[2 * q]);
      lf.col_perm.push_back(ao[2 * q + 1]);
    }
    c.kept_rows = read_ints(raw, PSG_LF_KEPT_ROWS, kd);
    c.kept_cols = read_ints(raw, PSG_LF_KEPT_COLS, kd);
    lf.core = std::move(c);
  }
  return lf;
}

// frame index -> row paired with it by the factorization (dense core)
std::vector<int> pairing(const LocalFactorization::DenseCore& dc) {
  std::vector<int> pr(dc.dim);
  for (int j = 0; j < dc.dim; ++j) pr[j] = j;
  for (const auto& [row, col] : dc.a_order) pr[col] = row;
  for (const auto& [row, col] : dc.b_order) pr[col] = row;
  for (std::size_t u = 0; u < dc.kept_cols.size(); ++u) pr[dc.kept_cols[u]] = dc.kept_rows[u];
  return pr;
}

const psg_local* dev_of(const LocalFactorization& lf) {
  if (!lf.device) fail(Errc::InvalidParameter, "local factorization has no device state");
  return lf.device.get();
}

// frame position of the reduced (kept) column u of a banded / cyclic core
int sep_frame(const LocalFactorization& lf, int u) { return u < lf.k0 ? u : lf.k0 + lf.L + (u - lf.k0); }

}  // namespace

// ---------------------------------------------------------------------------
// entry points (localfact.hpp:118-125)
// ---------------------------------------------------------------------------
LocalFactorization factor_lu(const PartitionBlock& M) { return run_factor(M, Strategy::Lu, 0.0); }
LocalFactorization factor_lud(const PartitionBlock& M) { return run_factor(M, Strategy::Lud, 0.0); }
LocalFactorization factor_cyclic_reduction(const PartitionBlock& M) {
  return run_factor(M, Strategy::CyclicReduction, 0.0);
}
LocalFactorization factor_arce(const PartitionBlock& M) { return run_factor(M, Strategy::Arce, 0.0); }
LocalFactorization factor_lu_pivot(const PartitionBlock& M, double tol) { return run_factor(M, Strategy::LuPivot, tol); }
LocalFactorization factor_qr(const PartitionBlock& M, double tol) { return run_factor(M, Strategy::Qr, tol); }

LocalFactorization factor(Strategy s, const PartitionBlock& M, double tol) {
  switch (s) {
    case Strategy::Lu:
    case Strategy::Lud:
    case Strategy::CyclicReduction:
    case Strategy::Arce: return run_factor(M, s, 0.0);
    case Strategy::LuPivot:
    case Strategy::Qr: return run_factor(M, s, tol);
  }
  fail(Errc::InvalidParameter, "unknown strategy");
}

// ---------------------------------------------------------------------------
// member operations (device)
// ---------------------------------------------------------------------------
void LocalFactorization::condense(const Vector& f_body, Vector& ghat, Vector& kept_rhs) const {
  if (int(f_body.size()) != L) fail(Errc::DimensionMismatch, "condense rhs length");
  ghat.assign(L, 0.0);
  kept_rhs.assign(kept_dim(), 0.0);
  char err[512];
  check(psg_local_condense(dev_of(*this), f_body.data(), ghat.data(), kept_rhs.data(), err, sizeof err), err);
}

Vector LocalFactorization::backsolve(const Vector& ghat, const Vector& x_kept) const {
  if (int(ghat.size()) != L || int(x_kept.size()) != kept_dim()) fail(Errc::DimensionMismatch, "backsolve lengths");
  Vector x(L);
  char err[512];
  check(psg_local_backsolve(dev_of(*this), ghat.data(), x_kept.data(), x.data(), err, sizeof err), err);
  return x;
}

Vector LocalFactorization::apply_N_inv(const Vector& rhs) const {
  if (int(rhs.size()) != L) fail(Errc::DimensionMismatch, "apply_N_inv length");
  Vector out(L);
  char err[512];
  check(psg_local_apply(dev_of(*this), 0, rhs.data(), out.data(), err, sizeof err), err);
  return out;
}

Vector LocalFactorization::apply_S_inv(const Vector& rhs) const {
  if (int(rhs.size()) != L) fail(Errc::DimensionMismatch, "apply_S_inv length");
  Vector out(L);
  char err[512];
  check(psg_local_apply(dev_of(*this), 1, rhs.data(), out.data(), err, sizeof err), err);
  return out;
}

// ---------------------------------------------------------------------------
// oracle materializations (host): F_loc, T_loc, G_loc of M^(i) = F T G
// ---------------------------------------------------------------------------
DenseMatrix LocalFactorization::dense_F_loc() const {
  const int dim = k0 + L + k1;
  if (const auto* bc = std::get_if<BandedCore>(&core)) {
    // body block N = unit lower factor (times the unit upper U' for Lud);
    // separator rows carry w^T / v^T
    DenseMatrix F = DenseMatrix::identity(dim);
    for (int i = 0; i < L; ++i)
      for (int q = 1; q <= std::min(bc->es, i); ++q) F.at(k0 + i, k0 + i - q) = bc->lent(i, bc->es - q);
    if (bc->unit_mid) {
      DenseMatrix Up = DenseMatrix::identity(L), Lo(L, L);
      for (int i = 0; i < L; ++i) {
        for (int j = 0; j < L; ++j) Lo.at(i, j) = F.at(k0 + i, k0 + j);
        for (int q = 1; q <= std::min(bc->er, L - 1 - i); ++q) Up.at(i, i + q) = bc->lent(i, bc->es + q) / bc->dvec[i + q];
      }
      const DenseMatrix N = matmul(Lo, Up);
      for (int i = 0; i < L; ++i)
        for (int j = 0; j < L; ++j) F.at(k0 + i, k0 + j) = N.at(i, j);
    }
    for (int x = 0; x < L; ++x) {
      for (int t = 0; t < k0; ++t) F.at(t, k0 + x) = w.at(x, t);
      for (int t = 0; t < k1; ++t) F.at(k0 + L + t, k0 + x) = v.at(x, t);
    }
    return F;
  }
  if (const auto* cc = std::get_if<CyclicCore>(&core)) {
    // F = E^{-1}, E the accumulated forward elimination operator
    const int g = cc->g;
    DenseMatrix E = DenseMatrix::identity(dim);
    auto block_rowop = [&](int tgt, int src, const DenseMatrix& Mb) {  // rows(tgt) -= Mb rows(src)
      for (int ti = 0; ti < g; ++ti)
        for (int j = 0; j < dim; ++j) {
          double acc = 0.0;
          for (int tj = 0; tj < g; ++tj) acc += Mb.at(ti, tj) * E.at(k0 + src * g + tj, j);
          E.at(k0 + tgt * g + ti, j) -= acc;
        }
    };
    for (const auto& e : cc->elims) {
      block_rowop(e.lnb, e.j, e.ml);
      block_rowop(e.rnb, e.j, e.mr);
    }
    const int rg = int(cc->rem.size()) * g;
    for (int u = 0; u < k0 + k1; ++u) {
      const int row = sep_frame(*this, u);
      for (int q = 0; q < rg; ++q) {
        const double mu = cc->rmat_d2inv.at(u, q);
        if (mu == 0.0) continue;
        const int src = k0 + cc->rem[q / g] * g + q % g;
        for (int j = 0; j < dim; ++j) E.at(row, j) -= mu * E.at(src, j);
      }
    }
    return inverse(E);
  }
  const auto& dc = std::get<DenseCore>(core);
  const std::vector<int> pr = pairing(dc);
  DenseMatrix F(dim, dim);
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < dim; ++j) F.at(i, j) = dc.Linv.at(i, pr[j]);
  return F;
}

namespace {

// the cyclic core's middle matrix: pivot blocks, their couplings, the
// remaining system and the separators' condensed rows
DenseMatrix cyclic_middle(const LocalFactorization& lf) {
  const auto& cc = std::get<LocalFactorization::CyclicCore>(lf.core);
  const int k0 = lf.k0, L = lf.L, kd = lf.k0 + lf.k1, dim = k0 + L + lf.k1, g = cc.g;
  DenseMatrix W(dim, dim);
  for (int u = 0; u < kd; ++u)
    for (int q = 0; q < kd; ++q) W.at(sep_frame(lf, u), sep_frame(lf, q)) = lf.kept.at(u, q);
  for (const auto& e : cc.elims) {
    const DenseMatrix piv = inverse(e.dinv);
    for (int ti = 0; ti < g; ++ti)
      for (int tj = 0; tj < g; ++tj) {
        W.at(k0 + e.j * g + ti, k0 + e.j * g + tj) = piv.at(ti, tj);
        W.at(k0 + e.j * g + ti, k0 + e.lnb * g + tj) = e.a.at(ti, tj);
        W.at(k0 + e.j * g + ti, k0 + e.rnb * g + tj) = e.c.at(ti, tj);
      }
  }
  const int R = int(cc.rem.size());
  for (int u = 0; u < R; ++u)
    for (int ti = 0; ti < g; ++ti) {
      const int row = k0 + cc.rem[u] * g + ti;
      for (int q = 0; q < R; ++q)
        for (int tj = 0; tj < g; ++tj) W.at(row, k0 + cc.rem[q] * g + tj) = cc.d2.at(u * g + ti, q * g + tj);
      for (int c = 0; c < kd; ++c) W.at(row, sep_frame(lf, c)) = cc.cmat.at(u * g + ti, c);
    }
  return W;
}

}  // namespace

DenseMatrix LocalFactorization::dense_T_loc() const {
  const int dim = k0 + L + k1;
  DenseMatrix T = DenseMatrix::identity(dim);
  if (const auto* dc = std::get_if<DenseCore>(&core)) {
    // kept columns: their paired rows of the middle matrix, restricted to kept columns
    for (std::size_t u = 0; u < dc->kept_cols.size(); ++u) {
      const int col = dc->kept_cols[u];
      for (int j = 0; j < dim; ++j) T.at(col, j) = 0.0;
      for (int kc : dc->kept_cols) T.at(col, kc) = dc->Wmid.at(dc->kept_rows[u], kc);
    }
    return T;
  }
  for (int u = 0; u < k0 + k1; ++u)
    for (int q = 0; q < k0 + k1; ++q) T.at(sep_frame(*this, u), sep_frame(*this, q)) = kept.at(u, q);
  return T;
}

DenseMatrix LocalFactorization::dense_G_loc() const {
  const int dim = k0 + L + k1;
  if (const auto* bc = std::get_if<BandedCore>(&core)) {
    DenseMatrix G = DenseMatrix::identity(dim);
    for (int i = 0; i < L; ++i) {
      if (bc->unit_mid)
        G.at(k0 + i, k0 + i) = bc->dvec[i];
      else
        for (int q = 0; q <= std::min(bc->er, L - 1 - i); ++q) G.at(k0 + i, k0 + i + q) = bc->lent(i, bc->es + q);
      for (int t = 0; t < k0; ++t) G.at(k0 + i, t) = z.at(i, t);
      for (int t = 0; t < k1; ++t) G.at(k0 + i, k0 + L + t) = y.at(i, t);
    }
    return G;
  }
  if (std::holds_alternative<CyclicCore>(core)) {
    DenseMatrix G = cyclic_middle(*this);
    for (int u = 0; u < k0 + k1; ++u) {
      const int row = sep_frame(*this, u);
      for (int j = 0; j < dim; ++j) G.at(row, j) = j == row ? 1.0 : 0.0;
    }
    return G;
  }
  const auto& dc = std::get<DenseCore>(core);
  const std::vector<int> pr = pairing(dc);
  DenseMatrix G(dim, dim);
  for (int c = 0; c < dim; ++c)
    for (int j = 0; j < dim; ++j) G.at(c, j) = dc.Wmid.at(pr[c], j);
  for (int kc : dc.kept_cols)
    for (int j = 0; j < dim; ++j) G.at(kc, j) = j == kc ? 1.0 : 0.0;
  if (dc.has_right) G = matmul(G, dc.Rinv);
  return G;
}

DenseMatrix LocalFactorization::dense_N() const {
  const DenseMatrix F = dense_F_loc();
  DenseMatrix N(L, L);
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j) N.at(i, j) = F.at(k0 + i, k0 + j);
  return N;
}

DenseMatrix LocalFactorization::dense_S() const {
  const DenseMatrix G = dense_G_loc();
  DenseMatrix S(L, L);
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j) S.at(i, j) = G.at(k0 + i, k0 + j);
  return S;
}

}  // namespace parsol
