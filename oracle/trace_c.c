/* CPU oracle helper — TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py cpu_baseline).
 *
 * Brute-force nearest hit over ALL primitives, restating src/scene.py:227-268
 * (2D cross-product segment test / 3D Möller–Trumbore in float64, inclusive
 * barycentrics, t > t_eps, first-min tie break = lowest primitive index), with the
 * rays split across OpenMP threads.  Same algorithm as the numpy oracle; compiled
 * with -ffp-contract=off so no FMA changes the float64 arithmetic.  Pinned against
 * the reference by tests/test_oracle_golden.py (golden rays from the reference).
 */
#include <math.h>
#include <stdint.h>

static inline double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
static inline void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

/* prim: K × 9 (v0, e1, e2) for dim 3, K × 4 (a, e) for dim 2. */
void oracle_trace(int dim, int64_t K, const double* prim, int64_t m, const double* orig,
                  const double* dirs, double t_eps, double* out_t, int64_t* out_idx, int n_threads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(n_threads)
  for (int64_t r = 0; r < m; ++r) {
    double best = INFINITY;
    int64_t bi = -1;
    if (dim == 3) {
      const double* o = orig + 3 * r;
      const double* d = dirs + 3 * r;
      for (int64_t k = 0; k < K; ++k) {
        const double* P = prim + 9 * k;
        double pv[3], tv[3], qv[3];
        cross3(d, P + 6, pv);
        double det = dot3(P + 3, pv);
        tv[0] = o[0] - P[0];
        tv[1] = o[1] - P[1];
        tv[2] = o[2] - P[2];
        double inv = 1.0 / det;
        double u = dot3(tv, pv) * inv;
        cross3(tv, P + 3, qv);
        double v = dot3(d, qv) * inv;
        double t = dot3(P + 6, qv) * inv;
        if (isfinite(t) && fabs(det) > 0.0 && u >= 0.0 && v >= 0.0 && u + v <= 1.0 && t > t_eps &&
            t < best) {
          best = t;
          bi = k;
        }
      }
    } else {
      const double* o = orig + 2 * r;
      const double* d = dirs + 2 * r;
      for (int64_t k = 0; k < K; ++k) {
        const double* P = prim + 4 * k;
        double ax = P[0] - o[0], ay = P[1] - o[1];
        double den = d[0] * P[3] - d[1] * P[2];
        double t = (ax * P[3] - ay * P[2]) / den;
        double u = (ax * d[1] - ay * d[0]) / den;
        if (fabs(den) > 0.0 && u >= 0.0 && u <= 1.0 && t > t_eps && t < best) {
          best = t;
          bi = k;
        }
      }
    }
    out_t[r] = best;
    out_idx[r] = bi;
  }
}
