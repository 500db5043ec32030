// parsol/structmat.hpp -- structured matrix descriptors (reference
// proj/include/parsol/structmat.hpp:11-78): the five kinds stored compactly in
// the reference layout, which the GPU kernels read in place.
//
// Difference: make() additionally accepts the Babd BVP layout s = m, r = 0
// (lower block bidiagonal rows + corner; BASELINE config 4) that the
// reference's make() rejects (src/structmat.cpp:173-174).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "parsol/dense.hpp"

namespace parsol {

enum class Kind { Banded, BlockTridiagonal, Abd, Babd, CirculantLike };

const char* kind_name(Kind k);
Kind kind_from_name(const std::string& s);

struct StructuredMatrix {
  Kind kind = Kind::Banded;
  int n = 0;
  int m = 1;
  int s = 0;
  int r = 0;
  std::vector<double> data;
  int corner_rows = 0;
  int corner_cols = 0;
  std::vector<double> corner;

  int block_count() const { return m > 0 ? n / m : 0; }
  double at(int i, int j) const;          ///< structural read, 0 outside the pattern
  bool in_structure(int i, int j) const;
  bool corner_canonical() const;
  bool operator==(const StructuredMatrix&) const = default;
};

StructuredMatrix make(Kind kind, int n, int m, int s, int r, std::vector<double> data,
                      std::vector<double> corner = {}, int corner_rows = 0, int corner_cols = 0);
std::size_t body_entry_count(Kind kind, int n, int m, int s, int r);
DenseMatrix to_dense(const StructuredMatrix& A, int limit = 2048);
/// y = A x on the GPU (fixed ascending-column order, no FMA: bit-identical to the reference).
Vector matvec(const StructuredMatrix& A, const Vector& x);
StructuredMatrix generate_random(Kind kind, int n, int m, int s, int r, std::uint64_t seed, double dominance);
std::pair<int, int> scalar_envelope(const StructuredMatrix& A);

}  // namespace parsol
