// parsol/seqref.hpp -- solve_sequential (reference proj/include/parsol/seqref.hpp:12).
// The B200 library has no CPU solver: this runs the GPU partition solver with
// an automatically chosen partition count (bodies of ~1023 rows).
#pragma once

#include "parsol/structmat.hpp"

namespace parsol {

Vector solve_sequential(const StructuredMatrix& A, const Vector& f);

}  // namespace parsol
