// Record finalisation on device: luminance Hessian → symmetric eigen → validity radii.
// Restates src/numerics.py:51-166 (closed-form 2×2, trigonometric 3×3 with gap and
// residual checks) and src/cache.py:59-91, :146-189.  The LAPACK `eigh` fallback of
// the reference is replaced by cyclic Jacobi (same eigenpairs up to sign/degenerate
// rotation; parity compares the quadratic form A·diag(R⁻²)·Aᵀ).
#pragma once

#include <cmath>

namespace vc {

template <int D>
__device__ inline void sort_by_abs(double* vals, double* V /* D×D row-major, columns = vectors */) {
  // stable sort of eigenpairs by descending |λ| (np.argsort(-|λ|, kind="stable"))
  int order[3] = {0, 1, 2};
  for (int i = 1; i < D; ++i) {
    int k = order[i];
    int j = i - 1;
    while (j >= 0 && fabs(vals[order[j]]) < fabs(vals[k])) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = k;
  }
  double v2[3], V2[9];
  for (int c = 0; c < D; ++c) {
    v2[c] = vals[order[c]];
    for (int r = 0; r < D; ++r) V2[r * D + c] = V[r * D + order[c]];
  }
  for (int c = 0; c < D; ++c) vals[c] = v2[c];
  for (int e = 0; e < D * D; ++e) V[e] = V2[e];
}

__device__ inline void eig2(const double* m, double* vals, double* V) {
  double a = m[0], b = m[1], c = m[3];
  double mean = 0.5 * (a + c), hd = 0.5 * (a - c);
  double disc = hypot(hd, b);
  vals[0] = mean + disc;
  vals[1] = mean - disc;
  if (disc <= 1e-14 * fmax(fabs(mean), 1e-300)) {
    V[0] = 1; V[1] = 0; V[2] = 0; V[3] = 1;
  } else {
    double v0 = hd + disc, v1 = b;
    double a0 = b, a1 = -hd + disc;
    if (a0 * a0 + a1 * a1 > v0 * v0 + v1 * v1) {
      v0 = a0;
      v1 = a1;
    }
    double nv = sqrt(v0 * v0 + v1 * v1);
    v0 /= nv;
    v1 /= nv;
    V[0] = v0; V[1] = -v1;
    V[2] = v1; V[3] = v0;
  }
  sort_by_abs<2>(vals, V);
}

__device__ inline double det3(const double* b) {
  return b[0] * (b[4] * b[8] - b[5] * b[7]) - b[1] * (b[3] * b[8] - b[5] * b[6]) +
         b[2] * (b[3] * b[7] - b[4] * b[6]);
}

// Returns false when the analytic solve is untrustworthy (src/numerics.py:76-124).
__device__ inline bool eig3_analytic(const double* m, double* vals, double* V) {
  double sc = 0.0;
  for (int e = 0; e < 9; ++e) sc = fmax(sc, fabs(m[e]));
  if (sc == 0.0) {
    for (int e = 0; e < 9; ++e) V[e] = (e % 4 == 0) ? 1.0 : 0.0;
    vals[0] = vals[1] = vals[2] = 0.0;
    return true;
  }
  double p1 = m[1] * m[1] + m[2] * m[2] + m[5] * m[5];
  if (p1 <= (1e-14 * sc) * (1e-14 * sc)) {
    for (int e = 0; e < 9; ++e) V[e] = (e % 4 == 0) ? 1.0 : 0.0;
    vals[0] = m[0];
    vals[1] = m[4];
    vals[2] = m[8];
    sort_by_abs<3>(vals, V);
    return true;
  }
  double q = (m[0] + m[4] + m[8]) / 3.0;
  double p2 = (m[0] - q) * (m[0] - q) + (m[4] - q) * (m[4] - q) + (m[8] - q) * (m[8] - q) + 2.0 * p1;
  double p = sqrt(p2 / 6.0);
  double Bm[9];
  for (int e = 0; e < 9; ++e) Bm[e] = (m[e] - ((e % 4 == 0) ? q : 0.0)) / p;
  double r = fmin(fmax(det3(Bm) / 2.0, -1.0), 1.0);
  double phi = acos(r) / 3.0;
  double hi = q + 2.0 * p * cos(phi);
  double lo = q + 2.0 * p * cos(phi + 2.0 * 3.141592653589793 / 3.0);
  vals[0] = hi;
  vals[1] = 3.0 * q - hi - lo;
  vals[2] = lo;
  double gap = fmin(fabs(vals[0] - vals[1]), fmin(fabs(vals[1] - vals[2]), fabs(vals[0] - vals[2])));
  if (gap < 1e-6 * sc) return false;
  for (int k = 0; k < 3; ++k) {
    double A[9];
    for (int e = 0; e < 9; ++e) A[e] = m[e] - ((e % 4 == 0) ? vals[k] : 0.0);
    double cs[3][3];
    const int rr[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    int best = 0;
    double bn = -1.0;
    for (int t = 0; t < 3; ++t) {
      const double* a = A + 3 * rr[t][0];
      const double* b = A + 3 * rr[t][1];
      cs[t][0] = a[1] * b[2] - a[2] * b[1];
      cs[t][1] = a[2] * b[0] - a[0] * b[2];
      cs[t][2] = a[0] * b[1] - a[1] * b[0];
      double nn = cs[t][0] * cs[t][0] + cs[t][1] * cs[t][1] + cs[t][2] * cs[t][2];
      if (nn > bn) {
        bn = nn;
        best = t;
      }
    }
    double nv = sqrt(bn);
    if (nv < 1e-12 * sc * sc) return false;
    for (int rw = 0; rw < 3; ++rw) V[rw * 3 + k] = cs[best][rw] / nv;
  }
  sort_by_abs<3>(vals, V);
  return true;
}

__device__ inline void eig3_jacobi(const double* m, double* vals, double* V) {
  double a[9];
  for (int e = 0; e < 9; ++e) {
    a[e] = m[e];
    V[e] = (e % 4 == 0) ? 1.0 : 0.0;
  }
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
    double diag = a[0] * a[0] + a[4] * a[4] + a[8] * a[8];
    if (off <= 1e-34 * diag || off == 0.0) break;
    const int PQ[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    for (int t = 0; t < 3; ++t) {
      int p = PQ[t][0], q = PQ[t][1];
      double apq = a[p * 3 + q];
      if (apq == 0.0) continue;
      double theta = (a[q * 3 + q] - a[p * 3 + p]) / (2.0 * apq);
      double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
      for (int k = 0; k < 3; ++k) {  // A ← Jᵀ A J
        double akp = a[k * 3 + p], akq = a[k * 3 + q];
        a[k * 3 + p] = c * akp - s * akq;
        a[k * 3 + q] = s * akp + c * akq;
      }
      for (int k = 0; k < 3; ++k) {
        double apk = a[p * 3 + k], aqk = a[q * 3 + k];
        a[p * 3 + k] = c * apk - s * aqk;
        a[q * 3 + k] = s * apk + c * aqk;
      }
      for (int k = 0; k < 3; ++k) {
        double vkp = V[k * 3 + p], vkq = V[k * 3 + q];
        V[k * 3 + p] = c * vkp - s * vkq;
        V[k * 3 + q] = s * vkp + c * vkq;
      }
    }
  }
  vals[0] = a[0];
  vals[1] = a[4];
  vals[2] = a[8];
  // eigh returns ascending order; then the stable |λ| sort
  int o[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i) {
    int k = o[i];
    int j = i - 1;
    while (j >= 0 && vals[o[j]] > vals[k]) {
      o[j + 1] = o[j];
      --j;
    }
    o[j + 1] = k;
  }
  double v2[3], V2[9];
  for (int c = 0; c < 3; ++c) {
    v2[c] = vals[o[c]];
    for (int r = 0; r < 3; ++r) V2[r * 3 + c] = V[r * 3 + o[c]];
  }
  for (int c = 0; c < 3; ++c) vals[c] = v2[c];
  for (int e = 0; e < 9; ++e) V[e] = V2[e];
  sort_by_abs<3>(vals, V);
}

// eigen_sym (src/numerics.py:127-166) for a symmetric D×D matrix m (row-major).
template <int D>
__device__ inline void eigen_sym(const double* m_in, double* vals, double* V) {
  double m[9];
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) m[r * D + c] = 0.5 * (m_in[r * D + c] + m_in[c * D + r]);
  double sc = 0.0;
  for (int e = 0; e < D * D; ++e) sc = fmax(sc, fabs(m[e]));
  if (sc == 0.0) {
    for (int e = 0; e < D * D; ++e) V[e] = (e % (D + 1) == 0) ? 1.0 : 0.0;
    for (int c = 0; c < D; ++c) vals[c] = 0.0;
    return;
  }
  for (int e = 0; e < D * D; ++e) m[e] /= sc;
  if constexpr (D == 2) {
    eig2(m, vals, V);
  } else {
    bool ok = eig3_analytic(m, vals, V);
    if (ok) {
      double nrm = 0.0, res = 0.0, gram = 0.0;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          double rc = 0.0, g = 0.0;
          for (int k = 0; k < 3; ++k) {
            rc += V[r * 3 + k] * vals[k] * V[c * 3 + k];
            g += V[k * 3 + r] * V[k * 3 + c];
          }
          double d = rc - m[r * 3 + c];
          res += d * d;
          nrm += m[r * 3 + c] * m[r * 3 + c];
          double gd = g - (r == c ? 1.0 : 0.0);
          gram += gd * gd;
        }
      if (sqrt(res) > 0.5e-6 * sqrt(nrm) || sqrt(gram) > 1e-10) ok = false;
    }
    if (!ok) eig3_jacobi(m, vals, V);
  }
  for (int c = 0; c < D; ++c) vals[c] *= sc;
}

}  // namespace vc
