/* Forcing g(t) for the IVP measurements (tools/ode_bench.py): thread-safe, as
 * the reference calls it from OpenMP workers.  ctx points at the dimension. */
#include <math.h>

void ode_forcing(double t, double* out, void* ctx) {
  const int m = *(const int*)ctx;
  for (int q = 0; q < m; ++q) out[q] = sin((q + 1) * t) + 0.5 * cos(2.0 * t);
}
