// qem_expfam.cu -- EMA over mean parameters + M-step for non-Gaussian Q families (NEXT row f1,
// DESIGN.md): Gamma, Beta, Bernoulli, Categorical.  "Exponential family distributions are
// completely determined by their mean parameters"; "a Beta's parameters are
// recovered from expectations of log transformations"; Alg. 1 lines 3 and 6.
//
//   Gamma(k, th)      m = (E z, E ln z) = (k/th, psi(k) - ln th):
//                     solve psi(k) - ln k = m2 - ln m1 for ln k (Newton), th = k / m1
//   Beta(a, b)        m = (E ln z, E ln(1-z)) = (psi(a) - psi(a+b), psi(b) - psi(a+b)):
//                     damped 2-d Newton in (ln a, ln b)
//   Dirichlet(a[C])   m = E ln z = psi(a) - psi(sum a): Newton with a Sherman-Morrison Hessian
//   Binomial(N, p)    m = E z = N p  (N given as C)
//   Multinomial(N, p) m = E z = N p  (p = m / sum m, as Categorical)
//   Bernoulli(p)      m = p
//   Categorical(p)    m = p (normalised)
// One thread per latent instance, fp64 throughout (digamma / trigamma by recurrence to x >= 8
// and their asymptotic series, ~1e-15 relative).
#include <math_constants.h>
#include <stdint.h>

#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

__device__ double digamma_d(double x) {
  double r = 0.0;
  while (x < 8.0) {
    r -= 1.0 / x;
    x += 1.0;
  }
  const double f = 1.0 / (x * x);
  // psi(x) ~ ln x - 1/(2x) - 1/(12x^2) + 1/(120x^4) - 1/(252x^6) + 1/(240x^8) - 1/(132x^10) + 691/(32760x^12)
  const double s =
      f * (-1.0 / 12 + f * (1.0 / 120 + f * (-1.0 / 252 + f * (1.0 / 240 + f * (-1.0 / 132 + f * (691.0 / 32760))))));
  return r + log(x) - 0.5 / x + s;
}

__device__ double trigamma_d(double x) {
  double r = 0.0;
  while (x < 8.0) {
    r += 1.0 / (x * x);
    x += 1.0;
  }
  const double f = 1.0 / (x * x);
  // psi'(x) ~ 1/x + 1/(2x^2) + 1/(6x^3) - 1/(30x^5) + 1/(42x^7) - 1/(30x^9) + 5/(66x^11) - 691/(2730x^13)
  const double s = f * (1.0 / 6 + f * (-1.0 / 30 + f * (1.0 / 42 + f * (-1.0 / 30 + f * (5.0 / 66 + f * (-691.0 / 2730))))));
  return r + 1.0 / x + 0.5 * f + s / x;
}

// Gamma shape from s = E ln z - ln E z (< 0): Newton on u = ln k for g(u) = psi(e^u) - u - s,
// g'(u) = k psi'(k) - 1 > 0.  Start: Minka's closed-form approximation.
__device__ int gamma_shape(double s, double& k) {
  if (!(s < 0.0)) return QEM_EXPFAM_INFEASIBLE;
  const double sp = -s;
  k = (3.0 - sp + sqrt((sp - 3.0) * (sp - 3.0) + 24.0 * sp)) / (12.0 * sp);
  double u = log(k);
  for (int it = 0; it < 60; ++it) {
    k = exp(u);
    const double g = digamma_d(k) - u - s;
    const double dg = k * trigamma_d(k) - 1.0;
    double step = g / dg;
    if (step > 2.0) step = 2.0;
    if (step < -2.0) step = -2.0;
    u -= step;
    // g' = k psi'(k) - 1 ~ 1/(2k) for large k, so rounding noise in g moves u by ~1e-16 |u| k:
    // stop at 1e-12 relative (k to ~1e-12), after one more polishing step
    if (fabs(step) < 1e-12 * fmax(1.0, fabs(u))) {
      k = exp(u);
      u -= (digamma_d(k) - u - s) / (k * trigamma_d(k) - 1.0);
      k = exp(u);
      return QEM_EXPFAM_OK;
    }
  }
  k = exp(u);
  return QEM_EXPFAM_NO_CONVERGENCE;
}

// Beta (a, b) from (m1, m2) = (E ln z, E ln(1-z)): damped Newton in (ln a, ln b).
__device__ int beta_params(double m1, double m2, double& a, double& b) {
  const double g1 = exp(m1), g2 = exp(m2);
  if (!(m1 < 0.0 && m2 < 0.0 && g1 + g2 < 1.0)) return QEM_EXPFAM_INFEASIBLE;
  // start from psi(x) ~ ln(x - 1/2): a ~ (1 - g2) / (2 (1 - g1 - g2)), b ~ (1 - g1) / (2 (1 - g1 - g2))
  double la = log(0.5 * (1.0 - g2) / (1.0 - g1 - g2)), lb = log(0.5 * (1.0 - g1) / (1.0 - g1 - g2));
  auto resid = [&](double xa, double xb, double& r1, double& r2) {
    const double A = exp(xa), B = exp(xb), s = digamma_d(A + B);
    r1 = digamma_d(A) - s - m1;
    r2 = digamma_d(B) - s - m2;
  };
  double r1, r2;
  resid(la, lb, r1, r2);
  for (int it = 0; it < 100; ++it) {
    const double A = exp(la), B = exp(lb), t = trigamma_d(A + B);
    const double j11 = A * (trigamma_d(A) - t), j12 = -B * t, j21 = -A * t, j22 = B * (trigamma_d(B) - t);
    const double det = j11 * j22 - j12 * j21;
    const double d1 = (r1 * j22 - r2 * j12) / det, d2 = (j11 * r2 - j21 * r1) / det;
    const double n0 = r1 * r1 + r2 * r2;
    double lam = 1.0, na = la, nb = lb, q1 = r1, q2 = r2;
    for (int h = 0; h < 30; ++h, lam *= 0.5) {  // halve until the residual decreases
      na = la - lam * d1;
      nb = lb - lam * d2;
      resid(na, nb, q1, q2);
      if (q1 * q1 + q2 * q2 < n0 || n0 == 0.0) break;
    }
    const double moved = fmax(fabs(na - la), fabs(nb - lb));
    la = na;
    lb = nb;
    r1 = q1;
    r2 = q2;
    if (moved < 1e-13 * fmax(1.0, fmax(fabs(la), fabs(lb))) || (r1 == 0.0 && r2 == 0.0)) break;
  }
  a = exp(la);
  b = exp(lb);
  return fmax(fabs(r1), fabs(r2)) < 1e-10 ? QEM_EXPFAM_OK : QEM_EXPFAM_NO_CONVERGENCE;
}

// Dirichlet (a_1..a_C) from m_c = E ln z_c = psi(a_c) - psi(a_0), a_0 = sum a: Newton in a with
// the Hessian diag(psi'(a_c)) - psi'(a_0) 11^T inverted by Sherman-Morrison (O(C)), halving the
// step until every a_c stays positive; start from a_0 = 1/(1 - sum e^m), a_c = a_0 e^m_c (Minka's
// moment start).  C <= QEM_DIRICHLET_MAX_C.
#define QEM_DIRICHLET_MAX_C 16
__device__ int dirichlet_params(const double* m, int C, double* a) {
  double se = 0.0;
  for (int c = 0; c < C; ++c) {
    if (!(m[c] < 0.0)) return QEM_EXPFAM_INFEASIBLE;
    se += exp(m[c]);
  }
  if (!(se < 1.0) || C > QEM_DIRICHLET_MAX_C) return QEM_EXPFAM_INFEASIBLE;
  double al[QEM_DIRICHLET_MAX_C], g[QEM_DIRICHLET_MAX_C], q[QEM_DIRICHLET_MAX_C];
  const double a0i = 1.0 / (1.0 - se);
  for (int c = 0; c < C; ++c) al[c] = a0i * exp(m[c]) + 1e-3;
  for (int it = 0; it < 200; ++it) {
    double a0 = 0.0;
    for (int c = 0; c < C; ++c) a0 += al[c];
    const double p0 = digamma_d(a0), z = -trigamma_d(a0);
    double gmax = 0.0, sgq = 0.0, siq = 0.0;
    for (int c = 0; c < C; ++c) {
      g[c] = digamma_d(al[c]) - p0 - m[c];
      q[c] = trigamma_d(al[c]);
      gmax = fmax(gmax, fabs(g[c]));
      sgq += g[c] / q[c];
      siq += 1.0 / q[c];
    }
    if (gmax < 1e-13) {
      for (int c = 0; c < C; ++c) a[c] = al[c];
      return QEM_EXPFAM_OK;
    }
    const double b = sgq / (1.0 / z + siq);
    double lamb = 1.0;
    for (int h = 0; h < 60; ++h, lamb *= 0.5) {
      bool ok = true;
      for (int c = 0; c < C; ++c) ok = ok && al[c] - lamb * (g[c] - b) / q[c] > 0.0;
      if (ok) break;
    }
    for (int c = 0; c < C; ++c) al[c] -= lamb * (g[c] - b) / q[c];
  }
  for (int c = 0; c < C; ++c) a[c] = al[c];
  return QEM_EXPFAM_NO_CONVERGENCE;
}

struct FamArgs {
  int family, S, C;
  int64_t n;
  double lam;
  const double* m_new;
  double* m_ema;
  double* params;
  int32_t* status;
};

__global__ void __launch_bounds__(128) k_mstep_family(FamArgs a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    double* m = a.m_ema + i * a.S;
    const double* mn = a.m_new + i * a.S;
    for (int s = 0; s < a.S; ++s) m[s] = a.lam * m[s] + (1.0 - a.lam) * mn[s];  // EMA over mean parameters
    double* p = a.params + i * a.S;
    int st = QEM_EXPFAM_OK;
    if (a.family == QEM_QFAMILY_GAMMA) {
      double k = CUDART_NAN;
      st = m[0] > 0.0 ? gamma_shape(m[1] - log(m[0]), k) : QEM_EXPFAM_INFEASIBLE;
      p[0] = k;
      p[1] = k / m[0];
    } else if (a.family == QEM_QFAMILY_BETA) {
      double x = CUDART_NAN, y = CUDART_NAN;
      st = beta_params(m[0], m[1], x, y);
      p[0] = x;
      p[1] = y;
    } else if (a.family == QEM_QFAMILY_BERNOULLI) {
      st = (m[0] >= 0.0 && m[0] <= 1.0) ? QEM_EXPFAM_OK : QEM_EXPFAM_INFEASIBLE;
      p[0] = fmin(fmax(m[0], 0.0), 1.0);
    } else if (a.family == QEM_QFAMILY_DIRICHLET) {
      st = dirichlet_params(m, a.C, p);
      if (st == QEM_EXPFAM_INFEASIBLE)
        for (int c = 0; c < a.C; ++c) p[c] = CUDART_NAN;
    } else if (a.family == QEM_QFAMILY_BINOMIAL) {  // m = E z = N p, C = N trials
      st = (m[0] >= 0.0 && m[0] <= a.C) ? QEM_EXPFAM_OK : QEM_EXPFAM_INFEASIBLE;
      p[0] = fmin(fmax(m[0] / a.C, 0.0), 1.0);
    } else {  // categorical / multinomial: m = E onehot(z) or E counts, p = m / sum m
      double tot = 0.0;
      for (int c = 0; c < a.C; ++c) tot += m[c];
      st = tot > 0.0 ? QEM_EXPFAM_OK : QEM_EXPFAM_INFEASIBLE;
      for (int c = 0; c < a.C; ++c) p[c] = m[c] / tot;
    }
    if (a.status) a.status[i] = st;
  }
}

cudaError_t launch_mstep_family(int family, int64_t n, int C, double lam, const double* m_new, double* m_ema,
                                double* params, int32_t* status, cudaStream_t st) {
  FamArgs a{};
  a.family = family;
  a.S = family == QEM_QFAMILY_GAMMA || family == QEM_QFAMILY_BETA
            ? 2
            : (family == QEM_QFAMILY_BERNOULLI || family == QEM_QFAMILY_BINOMIAL ? 1 : C);
  a.C = C;
  a.n = n;
  a.lam = lam;
  a.m_new = m_new;
  a.m_ema = m_ema;
  a.params = params;
  a.status = status;
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + 127) / 128;
  k_mstep_family<<<(unsigned)(blocks < 65535 * 8 ? blocks : 65535 * 8), 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace qem
