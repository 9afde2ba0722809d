/*
 * qem_oracle.c -- plain, slow, fp64 CPU oracle for the QEM MPIW E-step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2503_08264_b200/, include/qem.h) never links,
 * includes or calls anything here, and this file includes nothing from it.
 *
 * Every function below follows the paper (arXiv 2503.08264, PAPER.md under
 * /root/reference at survey time) step by step; citations are
 * "PAPER.md:<line> (<section / equation>)".
 *
 *  - The E-step is Eq. 7a-c (Sec. 3.2): an average over all
 *    K^n index tuples of r_k = P(x, z^k) / prod_i Q(z_i^{k_i}).  With a
 *    factorised Q and a tree-shaped model this sum factorises
 *    by distributivity over the plate structure (Limitations:
 *    "reduce the memory complexity from O(K^n)").  The functions below write
 *    that nested sum out directly: for every group and every parent index,
 *    a log-sum-exp over the child index (max pass, then sum-of-exp pass),
 *    groups summed in index order, then the root log-sum-exp.
 *  - Marginal weights of each latent are the normalised Eq. 7b weights summed
 *    over all other indices (Eq. 7a with m(z) = indicator of one sample).
 *  - Moments are E[T(z)] = (E z, E z^2) under those weights (PAPER.md:218,
 *    691-692; Eq. m_one(z)).
 *  - The QEM step is Algorithm 1: M-step from the mean
 *    parameters, z ~ Q_t, E-step, EMA over mean parameters (Eq. 9,
 *    PAPER.md:242-245) with the history-weight reading (R5).
 *
 * Readings of silent/ambiguous points (R1..R21) are listed in DESIGN.md.
 * Pins: tests/test_oracle.py check this file against literal K^n
 * enumeration (oracle/brute.py, independent numpy code), closed-form
 * conjugate posteriors (oracle/closed_form.py), textbook special cases and
 * invariants.  Philox4x32-10 is pinned by the published Random123
 * known-answer vectors (tests/golden/philox4x32_10_kat.txt).
 *
 * All arithmetic is fp64 and uses the C library (exp, log, log1p, lgamma).
 * The only fp32 operations are the two places where the paper's method
 * *decides* a value in the kernel's precision (R22): the fp32
 * rounding of Q's parameters and the fp32 sample z = fmaf(sqrtf(v), eps, m).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_LN2PI 1.8378770664093454835606594728112

/* ---------------------------------------------------------------- helpers */

/* log N(x; m, v), v = variance (R9). */
static double lnN(double x, double m, double v) {
  double r = x - m;
  return -0.5 * (ORC_LN2PI + log(v)) - 0.5 * r * r / v;
}

/* log Bernoulli(y; sigmoid(eta)) = y*eta - softplus(eta) (R12). */
static double log_bern_logit(double y, double eta) {
  double sp = (eta > 0 ? eta : 0.0) + log1p(exp(-fabs(eta)));
  return y * eta - sp;
}

/* log Poisson(y; exp(eta)) = y*eta - exp(eta) - lgamma(y+1) (R11). */
static double log_pois_log(double y, double eta) {
  return y * eta - exp(eta) - lgamma(y + 1.0);
}

/* log sum_k exp(a[k]) over n terms with stride; two passes (max, then sum). */
static double lse(const double* a, long n, long stride) {
  double mx = -INFINITY;
  for (long k = 0; k < n; ++k) if (a[k * stride] > mx) mx = a[k * stride];
  if (mx == -INFINITY) return -INFINITY;
  double s = 0.0;
  for (long k = 0; k < n; ++k) s += exp(a[k * stride] - mx);
  return mx + log(s);
}

/* ------------------------------------------------------- two-level models */
/*
 * Root group (one shared copy index k, R2 / PAPER.md:394
 * "grouping random variables together in the proposal"):
 *   mu[0..d-1] ~ N(pm, pv) each, and, if scale_kind != 0, s ~ N(pm, pv).
 *   Root dims R = d + (scale_kind != 0); order mu_0..mu_{d-1}, s.
 * Groups i < n:  z_i in R^d ~ N(mu, V I) with
 *   V = fixed_var (scale_kind 0), exp(2 s) (1: log-sigma), exp(s) (2: log-variance).
 * Observations j < J per group:
 *   obs_kind 1: x_ij ~ N(z_i, obs_var)            (d == 1; Radon-like)
 *   obs_kind 2: y_ij ~ Bernoulli(sigmoid(z_i . x_ij)), x_ij in {0,1}^d
 *               (MovieLens-like)
 */
typedef struct {
  int d;
  int scale_kind;
  double fixed_var;
  int obs_kind;
  double obs_var;
  long n;
  int J;
  double prior_mean, prior_var;
} orc_model2;

static double group_var(const orc_model2* m, double s) {
  if (m->scale_kind == 0) return m->fixed_var;
  if (m->scale_kind == 1) return exp(2.0 * s);
  return exp(s);
}

/* log p(x_i | z_i = column kc of z_i) summed over the group's observations. */
static double group_loglik(const orc_model2* m, long i, const double* zi /*[d][K]*/, int K, int kc,
                           const double* xg, const unsigned char* xb, const unsigned char* yb) {
  double ll = 0.0;
  if (m->obs_kind == 1) {
    for (int j = 0; j < m->J; ++j) ll += lnN(xg[i * m->J + j], zi[kc], m->obs_var);
  } else {
    for (int j = 0; j < m->J; ++j) {
      double eta = 0.0;
      const unsigned char* xij = xb + ((size_t)i * m->J + j) * m->d;
      for (int r = 0; r < m->d; ++r) eta += (double)xij[r] * zi[(size_t)r * K + kc];
      ll += log_bern_logit((double)yb[(size_t)i * m->J + j], eta);
    }
  }
  return ll;
}

/*
 * Forward half of the two-level E-step: the root factor
 *   f_root(k) = log p(root^k) - log q(root^k)
 * and the per-group plate messages (elimination of each group's own index,
 * PAPER.md:393)
 *   g_i(k) = log (1/K) sum_k' exp(B_i(k,k') + A_i(k')),
 *   B_i(k,k') = log p(z_i^k' | root^k),  A_i(k') = log p(x_i | z_i^k') - log q(z_i^k').
 * Arrays as in orc2_estep.
 */
void orc2_forward(const orc_model2* m, int K, const double* z_root, const double* z, const double* qr_m,
                  const double* qr_v, const double* q_m, const double* q_v, const double* xg,
                  const unsigned char* xb, const unsigned char* yb, double* f_root, double* g) {
  const int d = m->d, R = d + (m->scale_kind != 0);
  const long n = m->n;
  const double logK = log((double)K);
  for (int k = 0; k < K; ++k) {
    double f = 0.0;
    for (int r = 0; r < R; ++r) {
      double v = z_root[(size_t)r * K + k];
      f += lnN(v, m->prior_mean, m->prior_var) - lnN(v, qr_m[r], qr_v[r]);
    }
    f_root[k] = f;
  }
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    const double* zi = z + (size_t)i * d * K;
    double* A = (double*)malloc(sizeof(double) * K);
    double* t = (double*)malloc(sizeof(double) * K);
    for (int kc = 0; kc < K; ++kc) {
      double a = group_loglik(m, i, zi, K, kc, xg, xb, yb);
      for (int r = 0; r < d; ++r) a -= lnN(zi[(size_t)r * K + kc], q_m[i * d + r], q_v[i * d + r]);
      A[kc] = a;
    }
    for (int kp = 0; kp < K; ++kp) {
      double V = group_var(m, R > d ? z_root[(size_t)d * K + kp] : 0.0);
      for (int kc = 0; kc < K; ++kc) {
        double b = 0.0;
        for (int r = 0; r < d; ++r) b += lnN(zi[(size_t)r * K + kc], z_root[(size_t)r * K + kp], V);
        t[kc] = b + A[kc];
      }
      g[(size_t)i * K + kp] = lse(t, K, 1) - logK;
    }
    free(A);
    free(t);
  }
}

/*
 * Backward half: each group's marginal weights given the root weights
 *   w_i(k') = sum_k w_root(k) exp(B_i(k,k') + A_i(k') - log K - g_i(k))
 * (Eq. 7a with m = indicator of z_i^k'), and their moments (E z, E z^2).
 */
void orc2_backward(const orc_model2* m, int K, const double* z_root, const double* z, const double* q_m,
                   const double* q_v, const double* xg, const unsigned char* xb, const unsigned char* yb,
                   const double* w_root, const double* g, double* w, double* m1, double* m2) {
  const int d = m->d, R = d + (m->scale_kind != 0);
  const long n = m->n;
  const double logK = log((double)K);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    const double* zi = z + (size_t)i * d * K;
    double* A = (double*)malloc(sizeof(double) * K);
    for (int kc = 0; kc < K; ++kc) {
      double av = group_loglik(m, i, zi, K, kc, xg, xb, yb);
      for (int r = 0; r < d; ++r) av -= lnN(zi[(size_t)r * K + kc], q_m[i * d + r], q_v[i * d + r]);
      A[kc] = av;
    }
    for (int kc = 0; kc < K; ++kc) {
      double s = 0.0;
      for (int kp = 0; kp < K; ++kp) {
        double V = group_var(m, R > d ? z_root[(size_t)d * K + kp] : 0.0);
        double b = 0.0;
        for (int r = 0; r < d; ++r) b += lnN(zi[(size_t)r * K + kc], z_root[(size_t)r * K + kp], V);
        s += w_root[kp] * exp(b + A[kc] - logK - g[(size_t)i * K + kp]);
      }
      w[(size_t)i * K + kc] = s;
    }
    for (int r = 0; r < d; ++r) {
      double s1 = 0.0, s2 = 0.0;
      for (int kc = 0; kc < K; ++kc) {
        double v = zi[(size_t)r * K + kc];
        s1 += w[(size_t)i * K + kc] * v;
        s2 += w[(size_t)i * K + kc] * v * v;
      }
      m1[i * d + r] = s1;
      m2[i * d + r] = s2;
    }
    free(A);
  }
}

/*
 * One MPIW E-step on a two-level model (Eq. 7a-c).
 * Inputs (all arrays row-major, k fastest):
 *   z_root [R][K], z [n][d][K]       samples (fp32-representable values)
 *   qr_m, qr_v [R]; q_m, q_v [n][d]  factorised Gaussian Q (mean, variance)
 *   xg [n][J] (obs 1) or xb [n][J][d], yb [n][J] (obs 2)
 * Outputs:
 *   log_pe; w_root [K]; w [n][K]; g [n][K] (per-group messages
 *   g_i(k) = log (1/K) sum_k' exp(B_i(k,k') + A_i(k')));
 *   m1_root, m2_root [R]; m1, m2 [n][d]  (E z, E z^2).
 * Returns 0, or 1 if the evidence is degenerate (all terms -inf).
 */
int orc2_estep(const orc_model2* m, int K, const double* z_root, const double* z,
               const double* qr_m, const double* qr_v, const double* q_m, const double* q_v,
               const double* xg, const unsigned char* xb, const unsigned char* yb,
               double* log_pe, double* w_root, double* w, double* g,
               double* m1_root, double* m2_root, double* m1, double* m2) {
  const int d = m->d, R = d + (m->scale_kind != 0);
  const long n = m->n;
  const double logK = log((double)K);
  double* f_root = (double*)malloc(sizeof(double) * K);
  orc2_forward(m, K, z_root, z, qr_m, qr_v, q_m, q_v, xg, xb, yb, f_root, g);

  /* Plate product and root: a(k) = f_root(k) + sum_i g_i(k) (index order). */
  double* a = (double*)malloc(sizeof(double) * K);
  for (int k = 0; k < K; ++k) {
    double s = f_root[k];
    for (long i = 0; i < n; ++i) s += g[(size_t)i * K + k];
    a[k] = s;
  }
  double L = lse(a, K, 1);
  *log_pe = L - logK;
  int degenerate = (L == -INFINITY) || isnan(L);
  for (int k = 0; k < K; ++k) w_root[k] = degenerate ? NAN : exp(a[k] - L);

  for (int r = 0; r < R; ++r) {
    double s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < K; ++k) {
      double v = z_root[(size_t)r * K + k];
      s1 += w_root[k] * v;
      s2 += w_root[k] * v * v;
    }
    m1_root[r] = s1;
    m2_root[r] = s2;
  }
  (void)d;
  orc2_backward(m, K, z_root, z, q_m, q_v, xg, xb, yb, w_root, g, w, m1, m2);
  free(a);
  free(f_root);
  return degenerate;
}

/* ----------------------------------------------------- three-level model */
/*
 * Config-3 shape (Bus-like nesting):
 *   root (shared index k_r): g ~ N(pm,pv), beta[0..P-1] ~ N(pm,pv); R = 1+P.
 *   top  a < A:        u_a  ~ N(g, top_var)
 *   sub  b < B (of a): v_ab ~ N(u_a, sub_var), instance index ab = a*B + b
 *   obs  j < J:        y_abj ~ Poisson(exp(v_ab + beta . x_abj)), x_abj in R^P
 * Each latent instance carries its own copy index (R1).
 */
typedef struct {
  int A, B, J, P;
  double top_var, sub_var;
  double prior_mean, prior_var;
} orc_model3;

/*
 * One MPIW E-step on the three-level model, written as the nested sum
 *   Pe = (1/K) sum_kr r_root(kr) prod_a (1/K) sum_ka r_a(kr,ka)
 *          prod_b (1/K) sum_kab r_ab(ka,kab) r_obs(kab,kr)
 * (Eq. 7c, factorised by distributivity).
 * Inputs: z_root [R][K]; z_top [A][K]; z_sub [A*B][K]; Q params per latent
 * dim (qr_*[R], qt_*[A], qs_*[A*B]); x [A*B][J][P]; y [A*B][J].
 * Outputs: log_pe; w_root [K]; w_top [A][K]; w_sub [A*B][K];
 *          (m1, m2) per latent dim of every level.
 */
int orc3_estep(const orc_model3* m, int K, const double* z_root, const double* z_top,
               const double* z_sub, const double* qr_m, const double* qr_v, const double* qt_m,
               const double* qt_v, const double* qs_m, const double* qs_v, const double* x,
               const double* y, double* log_pe, double* w_root, double* w_top, double* w_sub,
               double* m1_root, double* m2_root, double* m1_top, double* m2_top, double* m1_sub,
               double* m2_sub) {
  const int A = m->A, B = m->B, J = m->J, P = m->P, R = 1 + P;
  const double logK = log((double)K);
  const size_t KK = (size_t)K * K;
  double* f_root = (double*)malloc(sizeof(double) * K);
  double* Mab = (double*)malloc(sizeof(double) * (size_t)A * B * KK);  /* [ab][ka][kr] */
  double* Ta = (double*)malloc(sizeof(double) * (size_t)A * KK);       /* [a][kr][ka] */
  double* ha = (double*)malloc(sizeof(double) * (size_t)A * K);        /* [a][kr] */
  double* Lab = (double*)malloc(sizeof(double) * KK);                  /* [kab][kr] */
  double* t = (double*)malloc(sizeof(double) * K);

  for (int k = 0; k < K; ++k) {
    double f = 0.0;
    for (int r = 0; r < R; ++r) {
      double v = z_root[(size_t)r * K + k];
      f += lnN(v, m->prior_mean, m->prior_var) - lnN(v, qr_m[r], qr_v[r]);
    }
    f_root[k] = f;
  }

  /* Sub-plate: M_ab(ka,kr) = lse_kab [F_ab(ka,kab) + L_ab(kab,kr)] - log K. */
  for (int a = 0; a < A; ++a) {
    for (int b = 0; b < B; ++b) {
      const size_t ab = (size_t)a * B + b;
      for (int kab = 0; kab < K; ++kab) {
        double v = z_sub[ab * K + kab];
        for (int kr = 0; kr < K; ++kr) {
          double ll = 0.0;
          for (int j = 0; j < J; ++j) {
            double eta = v;
            for (int p = 0; p < P; ++p) eta += z_root[(size_t)(1 + p) * K + kr] * x[(ab * J + j) * P + p];
            ll += log_pois_log(y[ab * J + j], eta);
          }
          Lab[(size_t)kab * K + kr] = ll;
        }
      }
      for (int ka = 0; ka < K; ++ka) {
        double u = z_top[(size_t)a * K + ka];
        for (int kr = 0; kr < K; ++kr) {
          for (int kab = 0; kab < K; ++kab) {
            double v = z_sub[ab * K + kab];
            double F = lnN(v, u, m->sub_var) - lnN(v, qs_m[ab], qs_v[ab]);
            t[kab] = F + Lab[(size_t)kab * K + kr];
          }
          Mab[ab * KK + (size_t)ka * K + kr] = lse(t, K, 1) - logK;
        }
      }
    }
  }
  /* Top plate: T_a(kr,ka) = lnN(u;g,top_var) - log q(u) + sum_b M_ab(ka,kr);
     h_a(kr) = lse_ka T_a - log K. */
  for (int a = 0; a < A; ++a) {
    for (int kr = 0; kr < K; ++kr) {
      double gk = z_root[kr];
      for (int ka = 0; ka < K; ++ka) {
        double u = z_top[(size_t)a * K + ka];
        double T = lnN(u, gk, m->top_var) - lnN(u, qt_m[a], qt_v[a]);
        for (int b = 0; b < B; ++b) T += Mab[((size_t)a * B + b) * KK + (size_t)ka * K + kr];
        Ta[(size_t)a * KK + (size_t)kr * K + ka] = T;
      }
      ha[(size_t)a * K + kr] = lse(Ta + (size_t)a * KK + (size_t)kr * K, K, 1) - logK;
    }
  }
  /* Root. */
  double* av = (double*)malloc(sizeof(double) * K);
  for (int kr = 0; kr < K; ++kr) {
    double s = f_root[kr];
    for (int a = 0; a < A; ++a) s += ha[(size_t)a * K + kr];
    av[kr] = s;
  }
  double L = lse(av, K, 1);
  *log_pe = L - logK;
  int degenerate = (L == -INFINITY) || isnan(L);
  for (int k = 0; k < K; ++k) w_root[k] = exp(av[k] - L);

  /* Backward.  W_a(kr,ka) = w_root(kr) exp(T_a(kr,ka) - log K - h_a(kr)). */
  double* W = (double*)malloc(sizeof(double) * KK);
  for (int a = 0; a < A; ++a) {
    for (int kr = 0; kr < K; ++kr)
      for (int ka = 0; ka < K; ++ka)
        W[(size_t)kr * K + ka] =
            w_root[kr] * exp(Ta[(size_t)a * KK + (size_t)kr * K + ka] - logK - ha[(size_t)a * K + kr]);
    for (int ka = 0; ka < K; ++ka) {
      double s = 0.0;
      for (int kr = 0; kr < K; ++kr) s += W[(size_t)kr * K + ka];
      w_top[(size_t)a * K + ka] = s;
    }
    /* w_ab(kab) = sum_{kr,ka} W_a(kr,ka) exp(F_ab(ka,kab) + L_ab(kab,kr) - log K - M_ab(ka,kr)). */
    for (int b = 0; b < B; ++b) {
      const size_t ab = (size_t)a * B + b;
      for (int kab = 0; kab < K; ++kab) {
        double v = z_sub[ab * K + kab];
        for (int kr = 0; kr < K; ++kr) {
          double ll = 0.0;
          for (int j = 0; j < J; ++j) {
            double eta = v;
            for (int p = 0; p < P; ++p) eta += z_root[(size_t)(1 + p) * K + kr] * x[(ab * J + j) * P + p];
            ll += log_pois_log(y[ab * J + j], eta);
          }
          Lab[(size_t)kab * K + kr] = ll;
        }
      }
      for (int kab = 0; kab < K; ++kab) {
        double v = z_sub[ab * K + kab];
        double s = 0.0;
        for (int kr = 0; kr < K; ++kr) {
          for (int ka = 0; ka < K; ++ka) {
            double u = z_top[(size_t)a * K + ka];
            double F = lnN(v, u, m->sub_var) - lnN(v, qs_m[ab], qs_v[ab]);
            s += W[(size_t)kr * K + ka] *
                 exp(F + Lab[(size_t)kab * K + kr] - logK - Mab[ab * KK + (size_t)ka * K + kr]);
          }
        }
        w_sub[ab * K + kab] = s;
      }
    }
  }
  /* Moments (E z, E z^2) per latent dim. */
  for (int r = 0; r < R; ++r) {
    double s1 = 0, s2 = 0;
    for (int k = 0; k < K; ++k) {
      double v = z_root[(size_t)r * K + k];
      s1 += w_root[k] * v;
      s2 += w_root[k] * v * v;
    }
    m1_root[r] = s1;
    m2_root[r] = s2;
  }
  for (int a = 0; a < A; ++a) {
    double s1 = 0, s2 = 0;
    for (int k = 0; k < K; ++k) {
      double v = z_top[(size_t)a * K + k];
      s1 += w_top[(size_t)a * K + k] * v;
      s2 += w_top[(size_t)a * K + k] * v * v;
    }
    m1_top[a] = s1;
    m2_top[a] = s2;
  }
  for (long ab = 0; ab < (long)A * B; ++ab) {
    double s1 = 0, s2 = 0;
    for (int k = 0; k < K; ++k) {
      double v = z_sub[ab * K + k];
      s1 += w_sub[ab * K + k] * v;
      s2 += w_sub[ab * K + k] * v * v;
    }
    m1_sub[ab] = s1;
    m2_sub[ab] = s2;
  }
  free(W);
  free(av);
  free(t);
  free(Lab);
  free(ha);
  free(Ta);
  free(Mab);
  free(f_root);
  return degenerate;
}

/* ------------------------------------------------------ QEM M-step + EMA */

/* History weight lambda_t (R5): fixed new-weight w -> 1 - w;
   schedule p in (0,1) -> 1 - t^{-p} (Theorem 1). */
double orc_lambda(int t, double new_weight, double p) {
  if (p > 0.0) return 1.0 - pow((double)t, -p);
  return 1.0 - new_weight;
}

/* EMA over mean parameters (Eq. 9; Alg. 1 line 6):
   m_t = lambda m_{t-1} + (1 - lambda) m_one, applied to (E z, E z^2). */
void orc_ema(long n, double lam, double* m1, double* m2, const double* m1_new, const double* m2_new) {
  for (long i = 0; i < n; ++i) {
    m1[i] = lam * m1[i] + (1.0 - lam) * m1_new[i];
    m2[i] = lam * m2[i] + (1.0 - lam) * m2_new[i];
  }
}

/* Gaussian M-step (Alg. 1 line 3): mean = m1,
   variance = m2 - m1^2, floored (R8); parameters rounded to fp32
   (R22).  Returns the number of clamped variances. */
long orc_mstep(long n, const double* m1, const double* m2, double floor_v, float* q_m, float* q_v) {
  long clamps = 0;
  for (long i = 0; i < n; ++i) {
    double v = m2[i] - m1[i] * m1[i];
    if (!(v >= floor_v)) {
      v = floor_v;
      ++clamps;
    }
    q_m[i] = (float)m1[i];
    q_v[i] = (float)v;
  }
  return clamps;
}

/* Location-scale sampling z = m + sqrt(v) eps (App. E;
   Alg. 1 line 4), evaluated in fp32 as fmaf(sqrtf(v), eps, m) (R22).
   z[i][k] for latent dim i (n of them) and sample k. */
void orc_sample(long n, int K, const float* q_m, const float* q_v, const float* eps, float* z) {
  for (long i = 0; i < n; ++i) {
    float s = sqrtf(q_v[i]);
    for (int k = 0; k < K; ++k) z[(size_t)i * K + k] = fmaf(s, eps[(size_t)i * K + k], q_m[i]);
  }
}

/* ------------------------------------------------------------ Philox RNG */
/* Philox4x32-10 (Salmon et al. 2011), written out from its definition:
   10 rounds of the two multiply-xor S-boxes with Weyl key schedule.
   Counter layout for sample k of latent (level, instance, dim) at iteration
   t:  ctr = {k >> 2, dim, instance, (level << 24) | (t & 0xffffff)},
   key = {seed lo, seed hi}.  The four outputs feed two Box-Muller pairs:
   k%4 in {0,1} uses (o0, o1), k%4 in {2,3} uses (o2, o3);
   u = ((x >> 9) + 0.5) * 2^-23 (exact in fp32);
   eps = sqrt(-2 ln u_a) * (k even ? cos : sin)(2 pi u_b). */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Standard-normal draws eps[dim][k] for one latent instance. */
void orc_normal_eps(uint64_t seed, uint32_t iter, uint32_t level, uint32_t instance, int ndim, int K,
                    double* eps) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const double PI = 3.14159265358979323846;
  for (int r = 0; r < ndim; ++r) {
    for (int k = 0; k < K; ++k) {
      uint32_t ctr[4] = {(uint32_t)(k >> 2), (uint32_t)r, instance, (level << 24) | (iter & 0xffffffu)};
      uint32_t o[4];
      orc_philox4x32_10(ctr, key, o);
      uint32_t xa = (k & 2) ? o[2] : o[0];
      uint32_t xb = (k & 2) ? o[3] : o[1];
      double ua = ((double)(xa >> 9) + 0.5) * (1.0 / 8388608.0);
      double ub = ((double)(xb >> 9) + 0.5) * (1.0 / 8388608.0);
      double rad = sqrt(-2.0 * log(ua));
      eps[(size_t)r * K + k] = (k & 1) ? rad * sin(2.0 * PI * ub) : rad * cos(2.0 * PI * ub);
    }
  }
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the OpenMP loops over groups (timing only: results do not depend on it --
   every group's sums are computed by one thread and combined in index order). */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
