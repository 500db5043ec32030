// parsol/parfact.hpp -- the drop-in solver API (reference
// proj/include/parsol/parfact.hpp:14-63): parallel_factor / solve /
// solve_reduced / residual, executed on the B200 through the C ABI psg.h.
//
// ParallelFactorization keeps the reference's plan / strategy / reduced
// metadata / kept_maps; the factor data lives on the device behind `device`.
// `locals` stays empty on the GPU path (the kernels factor every partition in
// place); materialize_locals() fills any range of it on request, each entry a
// device-computed LocalFactorization.  ReducedSystem::T is materialised when
// dim <= kDenseReducedLimit; ReducedSystem::device keeps the reduced system
// solvable on the GPU at any size.
#pragma once

#include <memory>
#include <vector>

#include "parsol/localfact.hpp"
#include "parsol/partition.hpp"

struct psg_handle;

namespace parsol {

constexpr int kDenseReducedLimit = 4096;

struct ReducedSystem {
  int q = 0;
  int dim = 0;
  std::vector<int> block_sizes;
  std::vector<int> positions;
  std::vector<int> offsets;
  DenseMatrix T;  ///< dense image (only when dim <= kDenseReducedLimit)
  bool has_corner = false;
  /// The factorization this system came from (set by parallel_factor, used by
  /// solve_reduced when T is not materialised; empty for hand-built systems).
  std::shared_ptr<psg_handle> device;
};

struct SolveStats {
  double factor_seconds = 0;
  double phase1_seconds = 0;
  double phase2_seconds = 0;
  double phase3_seconds = 0;
  long long reduced_ops = 0;
  double certificate = 0;  ///< GPU: max componentwise backward error of the separator rows
  int fallbacks = 0;       ///< GPU: exact re-solves after a rejected speculative interface
};

struct ParallelFactorization {
  PartitionPlan plan;
  Strategy strategy = Strategy::Lu;
  std::vector<LocalFactorization> locals;  ///< empty unless materialize_locals() filled it
  ReducedSystem reduced;
  bool permuted = false;
  Permutation row_perm;
  std::vector<std::vector<int>> kept_maps;
  double factor_seconds = 0;  ///< wall time of parallel_factor, device work included
  std::shared_ptr<psg_handle> device;  ///< device factorization (psg_factor)
  int n = 0;
};

ParallelFactorization parallel_factor(const StructuredMatrix& A, int p, Strategy strategy, double tol = 1e-8);
/// Direct solve of the reduced system (src/parfact.cpp:134-184).  With T
/// materialised: LU with partial pivoting of T on the device, bit-identical to
/// the reference (psg_dense_solve); otherwise the handle's device reduced solve.
Vector solve_reduced(const ReducedSystem& R, const Vector& rhs, SolveStats* stats = nullptr);
/// The handle's own reduced solve at any dim (partition method on the device).
Vector solve_reduced(const ParallelFactorization& F, const Vector& rhs, SolveStats* stats = nullptr);
Vector solve(const ParallelFactorization& F, const Vector& f, SolveStats* stats = nullptr);
/// Device-resident solve (device pointers, optional cudaStream_t as void*).
void solve_device(const ParallelFactorization& F, const double* f_dev, double* x_dev, SolveStats* stats = nullptr,
                  void* stream = nullptr);
double residual(const StructuredMatrix& A, const Vector& x, const Vector& f);
/// Fill F.locals[first-1 .. first-1+count) with the reference's per-partition
/// factorizations of A (extract_block + factor on the device); count < 0: to p.
void materialize_locals(ParallelFactorization& F, const StructuredMatrix& A, int first = 1, int count = -1,
                        double tol = 1e-8);

}  // namespace parsol
