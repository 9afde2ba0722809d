// qem_three_level.cu -- MPIW E-step for the three-level nested count model
// (config 3: root {g, beta} -> A top groups u_a -> B subgroups v_ab ->
// Poisson(exp(v_ab + beta . x)) observations), sm_100a, fp64 throughout.
//
// The observation factor couples the subgroup index k_ab with the ROOT index
// k_r (beta sits in the root group), so the elimination is a
// K x K x K contraction per subgroup:
//   L_ab(kab,kr) = sum_j log Pois(y_abj; exp(v^kab + beta^kr . x_abj))
//   F_ab(ka,kab) = log N(v^kab; u^ka, sub_var) - log q(v^kab)
//   M_ab(ka,kr)  = lse_kab [F_ab + L_ab] - log K
//   T_a(kr,ka)   = log N(u^ka; g^kr, top_var) - log q(u^ka) + sum_b M_ab(ka,kr)
//   h_a(kr)      = lse_ka T_a - log K
//   a(kr)        = f_root(kr) + sum_a h_a(kr);  log Pe = lse a - log K
// Backward: W_a(kr,ka) = w_root(kr) exp(T_a - log K - h_a(kr));
//   w_u_a(ka) = sum_kr W_a;  w_v_ab(kab) = sum_{kr,ka} W_a exp(F_ab + L_ab - log K - M_ab).
// Counts reach ~5e6 (R14), so every table is fp64.
// The whole model is a few million terms: launch-bound, replicas only.
#include "qem_device.cuh"
#include "qem_internal.h"

namespace qem {

struct THArgs {
  int A, B, J, P, K;
  double top_var, sub_var, prior_mean, prior_var;
  const float* z_root;
  const float* qr_m;
  const float* qr_v;
  const float* z_top;
  const float* qt_m;
  const float* qt_v;
  const float* z_sub;
  const float* qs_m;
  const float* qs_v;
  const float* x;    // [AB][J][P]
  const int32_t* y;  // [AB][J]
  float* w_root;
  double* m1_root;
  double* v_root;
  float* w_top;
  double* m1_top;
  double* v_top;
  float* w_sub;
  double* m1_sub;
  double* v_sub;
  double* log_pe;
  double* trace;
  int64_t trace_len;
  int t_host;
  ThreeLevelWs ws;
  Counters* cnt;
};

__device__ __forceinline__ double lnq(double z, float m, float v) { return lnN(z, (double)m, (double)v); }

// f_root(k) = log p(g, beta) - log q(g, beta)
__global__ void k3_root_prep(THArgs a) {
  const int R = 1 + a.P;
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    double f = 0.0;
    for (int r = 0; r < R; ++r) {
      const double v = a.z_root[r * a.K + k];
      f += lnN(v, a.prior_mean, a.prior_var) - lnq(v, a.qr_m[r], a.qr_v[r]);
    }
    a.ws.f_root[k] = f;
  }
}

// The two [ab][K][K] fp64 tables of the sub-plate contraction, one thread per entry e of each:
//   L_ab(kab, kr)  (e = (ab K + kab) K + kr): the Poisson observation term;
//   F_ab(ka, kab)  (e = (ab K + ka) K + kab): lnN(v_ab^kab; u_a^ka, sub_var) - log q(v_ab^kab)
// (the logarithms once per entry, not once per root sample; read by k3_msub AND k3_wlevels, so the
// backward's P_ab(kab | ka, kr) is built from the same operand as M_ab).
__global__ void k3_tables(THArgs a) {
  const int K = a.K;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)a.A * a.B * K * K;
  if (e >= tot) return;
  const int lo = (int)(e % K);
  const int mid = (int)((e / K) % K);
  const int64_t ab = e / ((int64_t)K * K);
  {  // L: kab = mid, kr = lo
    const double v = a.z_sub[ab * K + mid];
    double ll = 0.0;
    for (int j = 0; j < a.J; ++j) {
      double eta = v;
      const float* xj = a.x + (ab * a.J + j) * a.P;
      for (int p = 0; p < a.P; ++p) eta += (double)a.z_root[(1 + p) * K + lo] * (double)xj[p];
      const double y = (double)a.y[ab * a.J + j];
      ll += log_pois(y, eta, lgamma(y + 1.0));
    }
    a.ws.Lab[e] = ll;
  }
  {  // F: ka = mid, kab = lo
    const int aa = (int)(ab / a.B);
    const double v = a.z_sub[ab * K + lo];
    a.ws.Fab[e] = lnN(v, (double)a.z_top[(int64_t)aa * K + mid], a.sub_var) - lnq(v, a.qs_m[ab], a.qs_v[ab]);
  }
}

__global__ void k3_msub(THArgs a) {
  const int K = a.K;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)a.A * a.B * K * K;
  if (e >= tot) return;
  const int kr = (int)(e % K);
  const int ka = (int)((e / K) % K);
  const int64_t ab = e / ((int64_t)K * K);
  const double* L = a.ws.Lab + ab * K * K;
  const double* F = a.ws.Fab + (ab * K + ka) * K;
  double mx = -CUDART_INF;
  for (int kab = 0; kab < K; ++kab) mx = fmax(mx, F[kab] + L[(int64_t)kab * K + kr]);
  double s = 0.0;
  for (int kab = 0; kab < K; ++kab) s += exp(F[kab] + L[(int64_t)kab * K + kr] - mx);
  a.ws.Mab[ab * K * K + (int64_t)ka * K + kr] = mx + log(s) - log((double)K);
}

// T_a(kr, ka) and h_a(kr): one warp per (a, kr), lanes over ka (the B sub-plate messages of a
// column summed by its lane; max / sum by warp shuffles in a fixed order).
__global__ void k3_top(THArgs a) {
  const int K = a.K, lane = threadIdx.x & 31;
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= a.A * K) return;
  const int kr = e % K, aa = e / K;
  const double g = a.z_root[kr];
  double* T = a.ws.Ta + ((int64_t)aa * K + kr) * K;
  double mx = -CUDART_INF;
  for (int ka = lane; ka < K; ka += 32) {
    const double u = a.z_top[(int64_t)aa * K + ka];
    double t = lnN(u, g, a.top_var) - lnq(u, a.qt_m[aa], a.qt_v[aa]);
    for (int b = 0; b < a.B; ++b) t += a.ws.Mab[((int64_t)aa * a.B + b) * K * K + (int64_t)ka * K + kr];
    T[ka] = t;
    mx = fmax(mx, t);
  }
  mx = warp_max(mx);
  double s = 0.0;
  for (int ka = lane; ka < K; ka += 32) s += exp(T[ka] - mx);
  s = warp_sum(s);
  if (lane == 0) a.ws.ha[(int64_t)aa * K + kr] = mx + log(s) - log((double)K);
}

// Root: one block.
__global__ void k3_root(THArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* wsh = reinterpret_cast<double*>(smem);
  double* scratch = wsh + a.K;
  const int K = a.K, tid = threadIdx.x, R = 1 + a.P;
  double mx = -CUDART_INF;
  for (int k = tid; k < K; k += blockDim.x) {
    double s = a.ws.f_root[k];
    for (int aa = 0; aa < a.A; ++aa) s += a.ws.ha[(int64_t)aa * K + k];
    wsh[k] = s;
    mx = fmax(mx, s);
  }
  const double M = block_max(mx, scratch);
  double s = 0.0;
  for (int k = tid; k < K; k += blockDim.x) s += exp(wsh[k] - M);
  const double L = M + log(block_sum(s, scratch));
  for (int k = tid; k < K; k += blockDim.x) {
    const double w = exp(wsh[k] - L);
    wsh[k] = w;
    a.w_root[k] = (float)w;
  }
  if (tid == 0) {
    const double lp = L - log((double)K);
    *a.log_pe = lp;
    a.ws.red[0] = L;
    if (a.trace) {
      const int t = resolve_iter(a.t_host, &a.cnt->iter);
      const int64_t j = (int64_t)t - a.cnt->trace_base;
      if (j >= 0 && j < a.trace_len) a.trace[j] = lp;
    }
    if (!(L > -CUDART_INF)) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_DEGENERATE);
    if (isnan(L)) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
  }
  __syncthreads();
  const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int r = wid; r < R; r += nw) {
    double s1 = 0.0;
    for (int k = lane; k < K; k += 32) s1 += wsh[k] * (double)a.z_root[r * K + k];
    s1 = warp_sum(s1);
    double s2 = 0.0;
    for (int k = lane; k < K; k += 32) {
      const double dz = (double)a.z_root[r * K + k] - s1;
      s2 += wsh[k] * dz * dz;
    }
    s2 = warp_sum(s2);
    if (lane == 0) {
      a.m1_root[r] = s1;
      a.v_root[r] = s2;
    }
  }
}

// W_a(kr, ka) = w_root(kr) exp(T_a(kr,ka) - log K - h_a(kr)), in place over Ta.
__global__ void k3_wtop(THArgs a) {
  const int K = a.K;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)a.A * K * K) return;
  const int kr = (int)((e / K) % K);
  const int aa = (int)(e / ((int64_t)K * K));
  const double wr = (double)a.w_root[kr];
  a.ws.Ta[e] = wr * exp(a.ws.Ta[e] - log((double)K) - a.ws.ha[(int64_t)aa * K + kr]);
}

// w_u_a(ka) = sum_kr W_a(kr,ka); w_v_ab(kab) = sum_{kr,ka} W_a(kr,ka) exp(F + L - log K - M).
__global__ void k3_wlevels(THArgs a) {
  // one warp per output weight: top weights w_a(ka) = sum_kr W_a(kr, ka) (lanes over kr), sub
  // weights w_ab(kab) = sum_{ka, kr} W_a(kr, ka) P_ab(kab | ka, kr) (lanes over ka, loop over kr)
  const int K = a.K, lane = threadIdx.x & 31;
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t ntop = (int64_t)a.A * K;
  const int64_t nsub = (int64_t)a.A * a.B * K;
  if (e < ntop) {
    const int ka = (int)(e % K), aa = (int)(e / K);
    double s = 0.0;
    for (int kr = lane; kr < K; kr += 32) s += a.ws.Ta[((int64_t)aa * K + kr) * K + ka];
    s = warp_sum(s);
    if (lane == 0) a.w_top[e] = (float)s;
    return;
  }
  const int64_t f = e - ntop;
  if (f >= nsub) return;
  const int kab = (int)(f % K);
  const int64_t ab = f / K;
  const int aa = (int)(ab / a.B);
  const double logK = log((double)K);
  double s = 0.0;
  for (int ka = lane; ka < K; ka += 32) {
    const double F = a.ws.Fab[(ab * K + ka) * K + kab];  // the operand M_ab was built from (k3_tables)
    for (int kr = 0; kr < K; ++kr) {
      const double W = a.ws.Ta[((int64_t)aa * K + kr) * K + ka];
      s += W * exp(F + a.ws.Lab[(ab * K + kab) * K + kr] - logK - a.ws.Mab[ab * K * K + (int64_t)ka * K + kr]);
    }
  }
  s = warp_sum(s);
  if (lane == 0) a.w_sub[ab * K + kab] = (float)s;
}

// Moments (E z, Var z) of the top and sub levels from their weights (fp64).
__global__ void k3_moments(THArgs a) {
  const int K = a.K;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ntop = a.A, nsub = (int64_t)a.A * a.B;
  const float *w, *z;
  double *m1, *v;
  int64_t i;
  if (e < ntop) {
    i = e;
    w = a.w_top;
    z = a.z_top;
    m1 = a.m1_top;
    v = a.v_top;
  } else if (e < ntop + nsub) {
    i = e - ntop;
    w = a.w_sub;
    z = a.z_sub;
    m1 = a.m1_sub;
    v = a.v_sub;
  } else {
    return;
  }
  double s1 = 0.0;
  bool bad = false;
  for (int k = 0; k < K; ++k) {
    const double wk = w[i * K + k];
    bad |= isnan(wk);
    s1 += wk * (double)z[i * K + k];
  }
  double s2 = 0.0;
  for (int k = 0; k < K; ++k) {
    const double dz = (double)z[i * K + k] - s1;
    s2 += (double)w[i * K + k] * dz * dz;
  }
  m1[i] = s1;
  v[i] = s2;
  if (bad) atomicOr(&a.cnt->flags, (uint32_t)QEM_FLAG_NAN);
}

static THArgs make_args3(qem_ctx* c) {
  THArgs a{};
  const qem_model_desc& d = c->desc;
  a.A = (int)d.n;
  a.B = d.n_sub;
  a.J = d.n_obs;
  a.P = d.n_cov;
  a.K = d.K;
  a.top_var = d.top_var;
  a.sub_var = d.sub_var;
  a.prior_mean = d.prior_mean;
  a.prior_var = d.prior_var;
  const qem_level *r = &c->bufs.level[0], *t = &c->bufs.level[1], *s = &c->bufs.level[2];
  a.z_root = r->z;
  a.qr_m = r->q_mean;
  a.qr_v = r->q_var;
  a.z_top = t->z;
  a.qt_m = t->q_mean;
  a.qt_v = t->q_var;
  a.z_sub = s->z;
  a.qs_m = s->q_mean;
  a.qs_v = s->q_var;
  a.x = reinterpret_cast<const float*>(c->bufs.x);
  a.y = reinterpret_cast<const int32_t*>(c->bufs.y);
  a.w_root = r->w;
  a.m1_root = r->m1;
  a.v_root = r->v;
  a.w_top = t->w;
  a.m1_top = t->m1;
  a.v_top = t->v;
  a.w_sub = s->w;
  a.m1_sub = s->m1;
  a.v_sub = s->v;
  a.log_pe = c->bufs.log_pe;
  a.trace = c->in_iterate ? c->bufs.trace : nullptr;
  a.trace_len = c->bufs.trace_len;
  a.t_host = 0;
  a.ws = c->th;
  a.cnt = c->cnt;
  return a;
}

static unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t th_forward(qem_ctx* c, cudaStream_t st) {
  THArgs a = make_args3(c);
  const int64_t KK = (int64_t)a.K * a.K, AB = (int64_t)a.A * a.B;
  k3_root_prep<<<1, 256, 0, st>>>(a);
  k3_tables<<<nblk(AB * KK, 128), 128, 0, st>>>(a);
  k3_msub<<<nblk(AB * KK, 128), 128, 0, st>>>(a);
  k3_top<<<nblk((int64_t)a.A * a.K * 32, 256), 256, 0, st>>>(a);
  c->launches += 4;
  return cudaGetLastError();
}

cudaError_t th_backward(qem_ctx* c, cudaStream_t st) {
  THArgs a = make_args3(c);
  const int64_t KK = (int64_t)a.K * a.K, AB = (int64_t)a.A * a.B;
  int nt = (a.K + 31) & ~31;
  if (nt < 32) nt = 32;
  k3_root<<<1, nt, (size_t)(a.K + 32) * sizeof(double), st>>>(a);
  k3_wtop<<<nblk((int64_t)a.A * KK, 128), 128, 0, st>>>(a);
  k3_wlevels<<<nblk(((int64_t)a.A * a.K + AB * a.K) * 32, 256), 256, 0, st>>>(a);
  k3_moments<<<nblk(a.A + AB, 64), 64, 0, st>>>(a);
  c->launches += 4;
  return cudaGetLastError();
}

}  // namespace qem
