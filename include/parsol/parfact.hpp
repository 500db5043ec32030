// parsol/parfact.hpp -- the drop-in solver API (reference
// proj/include/parsol/parfact.hpp:14-63): parallel_factor / solve /
// solve_reduced / residual, executed on the B200 through the C ABI psg.h.
//
// ParallelFactorization keeps the reference's plan / strategy / reduced
// metadata / kept_maps; the factor data lives on the device behind `device`.
// `locals` is not materialised on the GPU path, and ReducedSystem::T is
// materialised only when dim <= kDenseReducedLimit.
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
  ReducedSystem reduced;
  bool permuted = false;
  Permutation row_perm;
  std::vector<std::vector<int>> kept_maps;
  double factor_seconds = 0;
  std::shared_ptr<psg_handle> device;  ///< device factorization (psg_factor)
  int n = 0;
};

ParallelFactorization parallel_factor(const StructuredMatrix& A, int p, Strategy strategy, double tol = 1e-8);
Vector solve_reduced(const ParallelFactorization& F, const Vector& rhs, SolveStats* stats = nullptr);
Vector solve(const ParallelFactorization& F, const Vector& f, SolveStats* stats = nullptr);
/// Device-resident solve (device pointers, optional cudaStream_t as void*).
void solve_device(const ParallelFactorization& F, const double* f_dev, double* x_dev, SolveStats* stats = nullptr,
                  void* stream = nullptr);
double residual(const StructuredMatrix& A, const Vector& x, const Vector& f);

}  // namespace parsol
