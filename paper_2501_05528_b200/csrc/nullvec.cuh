// Null vector of one tagging-row subset, shared by the host planner
// (ublr_null_vectors, capi.cu) and its device twin (ublr_null_vectors_device,
// tagaspect.cu) so that both produce the same bits.
//
// ref/tagging.py:126-139 via ref/linalg.py:72-94: the last column of the
// complete Householder Q of A = T[rows]^T (ell x sz), LAPACK dgeqr2
// convention (v_0 = 1, beta = -sign(alpha) ||x||, tau = (beta - alpha) / beta),
// q = H_0 H_1 ... H_{sz-1} e_{ell-1}; plus the residual ||T[rows] q||.
// Every product and sum is explicitly rounded (no FMA contraction on the
// device, none available to the host compiler), and sqrt / division are
// correctly rounded on both sides, hence bitwise-equal results.
#pragma once
#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define UBLR_NV_HD __host__ __device__ __forceinline__
#else
#define UBLR_NV_HD inline
#endif

namespace ublr {
namespace nullvec {

#ifdef __CUDA_ARCH__
UBLR_NV_HD double mul(double a, double b) { return __dmul_rn(a, b); }
UBLR_NV_HD double add(double a, double b) { return __dadd_rn(a, b); }
UBLR_NV_HD double sub(double a, double b) { return __dsub_rn(a, b); }
UBLR_NV_HD double div(double a, double b) { return __ddiv_rn(a, b); }
UBLR_NV_HD double sqrt_(double a) { return __dsqrt_rn(a); }
#else
UBLR_NV_HD double mul(double a, double b) { return a * b; }
UBLR_NV_HD double add(double a, double b) { return a + b; }
UBLR_NV_HD double sub(double a, double b) { return a - b; }
UBLR_NV_HD double div(double a, double b) { return a / b; }
UBLR_NV_HD double sqrt_(double a) { return std::sqrt(a); }
#endif

constexpr int MAX_ELL = 32;

// A: ell x sz work matrix, column-major (A[i + j * ell] = T[rows[j]][i]),
// overwritten; tau: sz scratch; z: ell outputs. Returns the residual.
UBLR_NV_HD double null_vector(const double* T, int ell, const int32_t* rows, int sz, double* A, double* tau,
                              double* z) {
  for (int j = 0; j < sz; ++j)
    for (int i = 0; i < ell; ++i) A[i + j * ell] = T[(int64_t)rows[j] * ell + i];
  for (int j = 0; j < sz; ++j) tau[j] = 0.0;
  for (int j = 0; j < sz; ++j) {
    double* col = &A[j * ell];
    const double alpha = col[j];
    double ss = 0.0, scale = 0.0;
    for (int i = j + 1; i < ell; ++i) scale = fmax(scale, fabs(col[i]));
    if (scale > 0.0) {
      const double inv_scale = div(1.0, scale);   // dnrm2-style scaling, one division per column
      for (int i = j + 1; i < ell; ++i) {
        const double x = mul(col[i], inv_scale);
        ss = add(ss, mul(x, x));
      }
    }
    const double xnorm = mul(scale, sqrt_(ss));
    if (xnorm == 0.0) {
      tau[j] = 0.0;
      continue;
    }
    // dlapy2: w sqrt(1 + (z / w)^2), w = max(|alpha|, xnorm)
    const double aa = fabs(alpha), wmax = fmax(aa, xnorm), zmin = fmin(aa, xnorm);
    const double ratio = div(zmin, wmax);
    const double beta = -copysign(mul(wmax, sqrt_(add(1.0, mul(ratio, ratio)))), alpha);
    tau[j] = div(sub(beta, alpha), beta);
    const double inv = div(1.0, sub(alpha, beta));
    for (int i = j + 1; i < ell; ++i) col[i] = mul(col[i], inv);
    col[j] = beta;
    // H_j = I - tau v v^T (v = [1, col[j+1:]]) on the remaining columns
    for (int c = j + 1; c < sz; ++c) {
      double* a = &A[c * ell];
      double w = a[j];
      for (int i = j + 1; i < ell; ++i) w = add(w, mul(col[i], a[i]));
      w = mul(w, tau[j]);
      a[j] = sub(a[j], w);
      for (int i = j + 1; i < ell; ++i) a[i] = sub(a[i], mul(w, col[i]));
    }
  }
  for (int i = 0; i < ell; ++i) z[i] = (i == ell - 1) ? 1.0 : 0.0;
  for (int j = sz - 1; j >= 0; --j) {
    const double* v = &A[j * ell];
    double w = z[j];
    for (int i = j + 1; i < ell; ++i) w = add(w, mul(v[i], z[i]));
    w = mul(w, tau[j]);
    z[j] = sub(z[j], w);
    for (int i = j + 1; i < ell; ++i) z[i] = sub(z[i], mul(w, v[i]));
  }
  double r2 = 0.0;
  for (int j = 0; j < sz; ++j) {
    const double* t = T + (int64_t)rows[j] * ell;
    double d = 0.0;
    for (int i = 0; i < ell; ++i) d = add(d, mul(t[i], z[i]));
    r2 = add(r2, mul(d, d));
  }
  return sqrt_(r2);
}

}  // namespace nullvec
}  // namespace ublr
