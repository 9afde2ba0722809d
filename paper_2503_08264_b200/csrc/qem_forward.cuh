// qem_forward.cuh -- K2: fused unary terms + pair-tile forward log-sum-exp for
// two-level models (included by qem_two_level.cu; needs TLArgs, pad4, inv_fact).
//
// Per group i (one CTA at a time, persistent grid):
//  prep   columns k': A_i(k') = loglik - log q (fp64), u = z - mu_ref, |u|^2,
//         t_i(k') = B(k_ref,k') + A_i(k') (fp64), c_i = lse t_i - log K,
//         P_i = softmax t_i (fp32 in SMEM), ln P_i (-> HBM for the backward).
//  tile   rows k (registers, sorted by coefficient magnitude so a warp's rows
//         share a mode): dg_i(k) = log sum_k' P_i(k') exp(D_k(k')), by
//           mode 0: log1p(sum P expm1_5(D))   bound(|D|) <= 1/16
//           mode 1: log1p(sum P expm1_9(D))   bound(|D|) <= 1/2
//           mode 2: single-pass online log-sum-exp of D + ln P (ex2 on the SFU)
//         The mode is warp-uniform (max over the warp's rows).
#pragma once
// (included inside namespace qem)

template <int D>
struct FwdLayout {
  static constexpr int CS = pad4(D + 3);  // u[D], U2, P, lnP
  static constexpr int CH = 4;            // column chunk of the online log-sum-exp
  __host__ __device__ static int kpad(int K) { return (K + CH - 1) / CH * CH; }
  __host__ __device__ static size_t bytes(int K, int J) {
    size_t b = (size_t)kpad(K) * CS * sizeof(float);  // col
    b += (size_t)K * sizeof(double);                  // tref
    b += 32 * sizeof(double);                         // scratch
    b += 3 * QEM_MAX_D * sizeof(double);              // qconst
    b += 4 * sizeof(double);                          // obs stats
    b += (size_t)(2 * J + 4) * sizeof(uint32_t);      // bern masks + y
    return b;
  }
};

template <int D, int RP>
__device__ __forceinline__ float2 pair_D(const float2 (&al)[RP], const float2 (&ga)[RP], const float2 (&cc)[RP][D],
                                         int p, const float* u, float U2) {
  if constexpr (D == 1) {
    return fma2(fma2(ga[p], f2(u[0]), cc[p][0]), f2(u[0]), al[p]);
  } else {
    // two accumulators halve the dependent FMA chain
    float2 a0 = fma2(ga[p], f2(U2), al[p]);
    float2 a1 = mul2(cc[p][0], f2(u[0]));
#pragma unroll
    for (int r = 1; r < D; ++r) {
      if (r & 1)
        a0 = fma2(cc[p][r], f2(u[r]), a0);
      else
        a1 = fma2(cc[p][r], f2(u[r]), a1);
    }
    return add2(a0, a1);
  }
}

template <int D>
__device__ __forceinline__ void load_col(const float* cr, float (&u)[D], float& U2, float& P, float& lnP) {
  constexpr int CS = pad4(D + 3);
  float buf[CS];
#pragma unroll
  for (int q = 0; q < CS / 4; ++q) {
    const float4 v = reinterpret_cast<const float4*>(cr)[q];
    buf[4 * q] = v.x;
    buf[4 * q + 1] = v.y;
    buf[4 * q + 2] = v.z;
    buf[4 * q + 3] = v.w;
  }
#pragma unroll
  for (int r = 0; r < D; ++r) u[r] = buf[r];
  U2 = buf[D];
  P = buf[D + 1];
  lnP = buf[D + 2];
}

__device__ __forceinline__ float2 max2(float2 a, float2 b) { return make_float2(fmaxf(a.x, b.x), fmaxf(a.y, b.y)); }

template <int D, int RP, int N>
__device__ __forceinline__ void tile_poly(const float* col, int Kp, const float2 (&al)[RP], const float2 (&ga)[RP],
                                          const float2 (&cc)[RP][D], float (&dgv)[2 * RP]) {
  constexpr int CS = pad4(D + 3);
  float2 acc[RP];
#pragma unroll
  for (int p = 0; p < RP; ++p) acc[p] = f2(0.f);
#pragma unroll 2
  for (int kc = 0; kc < Kp; ++kc) {
    float u[D], U2, P, lnP;
    load_col<D>(col + (size_t)kc * CS, u, U2, P, lnP);
#pragma unroll
    for (int p = 0; p < RP; ++p) acc[p] = fma2(f2(P), expm1_poly<N>(pair_D<D, RP>(al, ga, cc, p, u, U2)), acc[p]);
  }
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    dgv[2 * p] = log1pf(acc[p].x);
    dgv[2 * p + 1] = log1pf(acc[p].y);
  }
}

template <int D, int RP>
__device__ __forceinline__ void tile_online(const float* col, int Kp, const float2 (&al)[RP], const float2 (&ga)[RP],
                                            const float2 (&cc)[RP][D], float (&dgv)[2 * RP]) {
  constexpr int CS = pad4(D + 3);
  constexpr int CH = FwdLayout<D>::CH;
  float2 mr[RP], ac[RP];
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    mr[p] = f2(-CUDART_INF_F);
    ac[p] = f2(0.f);
  }
  for (int kc0 = 0; kc0 < Kp; kc0 += CH) {
    float2 tv[CH][RP];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      float u[D], U2, P, lnP;
      load_col<D>(col + (size_t)(kc0 + c) * CS, u, U2, P, lnP);
#pragma unroll
      for (int p = 0; p < RP; ++p) tv[c][p] = add2(pair_D<D, RP>(al, ga, cc, p, u, U2), f2(lnP));
    }
#pragma unroll
    for (int p = 0; p < RP; ++p) {
      float2 cm = tv[0][p];
#pragma unroll
      for (int c = 1; c < CH; ++c) cm = max2(cm, tv[c][p]);
      const float2 mn = max2(mr[p], cm);
      const float2 sc = make_float2(ex2((mr[p].x - mn.x) * kLog2e), ex2((mr[p].y - mn.y) * kLog2e));
      const float2 nm = make_float2(-mn.x * kLog2e, -mn.y * kLog2e);
      float2 s = mul2(ac[p], sc);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const float2 e = fma2(tv[c][p], f2(kLog2e), nm);
        s = add2(s, make_float2(ex2(e.x), ex2(e.y)));
      }
      ac[p] = s;
      mr[p] = mn;
    }
  }
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    dgv[2 * p] = mr[p].x + logf(ac[p].x);
    dgv[2 * p + 1] = mr[p].y + logf(ac[p].y);
  }
}

// One CTA processes groups i = blockIdx.x, += gridDim.x.  Thread t owns the
// row slots s = 2(t*RP+p)+h (p < RP float2 pairs), i.e. rows k = perm[s];
// the row coefficients stay in registers for the whole kernel (they depend
// only on the root samples).  Column data (u, |u|^2, P, ln P) of the current
// group sit in shared memory and are read as warp-broadcasts.
template <int D, int OBS, int RP>
__global__ void __launch_bounds__(256) k_forward(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int CS = pad4(D + 3);
  constexpr int CW = D + 2;
  const int K = a.K, J = a.J, tid = threadIdx.x, NT = blockDim.x;
  const int Kp = FwdLayout<D>::kpad(K);
  float* col = reinterpret_cast<float*>(smem);
  double* tref = reinterpret_cast<double*>(col + (size_t)Kp * CS);
  double* scratch = tref + K;
  double* qconst = scratch + 32;  // [3][QEM_MAX_D]
  double* ostat = qconst + 3 * QEM_MAX_D;
  uint32_t* bmask = reinterpret_cast<uint32_t*>(ostat + 4);
  uint32_t* ybits = bmask + J;

  const RefInfo ref = *a.ws.ref;
  // Row coefficients in registers.
  float2 al[RP], ga[RP], cc[RP][D];
  float rb_a[2 * RP], rb_g[2 * RP], rb_c[2 * RP];
  int kid[2 * RP];
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    float av[2], gv[2], cv[2][D];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * (tid * RP + p) + h;  // a warp owns a contiguous run of sorted slots
      const bool ok = s < K;
      const int k = ok ? a.ws.perm[s] : 0;
      kid[2 * p + h] = ok ? k : -1;
      const float* fc = a.ws.fwd_coef + (size_t)k * CW;
      av[h] = ok ? fc[0] : 0.f;
      gv[h] = ok ? fc[1] : 0.f;
      float cn = 0.f;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        cv[h][r] = ok ? fc[2 + r] : 0.f;
        cn = fmaf(cv[h][r], cv[h][r], cn);
      }
      rb_a[2 * p + h] = fabsf(av[h]);
      rb_g[2 * p + h] = fabsf(gv[h]);
      rb_c[2 * p + h] = sqrtf(cn);
    }
    al[p] = make_float2(av[0], av[1]);
    ga[p] = make_float2(gv[0], gv[1]);
#pragma unroll
    for (int r = 0; r < D; ++r) cc[p][r] = make_float2(cv[0][r], cv[1][r]);
  }
  double G[2 * RP];
#pragma unroll
  for (int j = 0; j < 2 * RP; ++j) G[j] = 0.0;
  double csum = 0.0;
  const double logK = log((double)K);
  // padding columns contribute nothing: P = 0, ln P = -inf
  for (int kc = K + tid; kc < Kp; kc += NT) {
    float* cp = col + (size_t)kc * CS;
    for (int r = 0; r < CS; ++r) cp[r] = 0.f;
    cp[D + 2] = -CUDART_INF_F;
  }

  for (int64_t i = blockIdx.x; i < a.n_local; i += gridDim.x) {
    __syncthreads();
    // ---- per-group constants: Q_i (log q) and observation summaries
    if (tid < D) {
      const double m = a.q_m[i * D + tid], v = a.q_v[i * D + tid];
      qconst[tid] = m;
      qconst[QEM_MAX_D + tid] = 0.5 / v;
      qconst[2 * QEM_MAX_D + tid] = -0.5 * (kLn2Pi + log(v));
    }
    if constexpr (OBS == QEM_OBS_GAUSS) {
      if (tid < 32) {
        const float* x = reinterpret_cast<const float*>(a.x) + i * J;
        double sx = 0.0, sxx = 0.0;
        for (int j = tid; j < J; j += 32) {
          const double xv = x[j];
          sx += xv;
          sxx += xv * xv;
        }
        sx = warp_sum(sx);
        sxx = warp_sum(sxx);
        if (tid == 0) {
          ostat[0] = sx;
          ostat[1] = sxx;
          ostat[2] = -0.5 * J * (kLn2Pi + log(a.obs_var));
          ostat[3] = 0.5 / a.obs_var;
        }
      }
    } else {
      const uint8_t* x = reinterpret_cast<const uint8_t*>(a.x) + (size_t)i * J * D;
      const uint8_t* y = reinterpret_cast<const uint8_t*>(a.y) + (size_t)i * J;
      for (int j = tid; j < J; j += NT) {
        uint32_t mk = 0;
#pragma unroll
        for (int r = 0; r < D; ++r) mk |= (x[j * D + r] ? 1u : 0u) << r;
        bmask[j] = mk;
        ybits[j] = y[j] ? 1u : 0u;
      }
    }
    __syncthreads();
    // ---- unary terms A_i(k') (fp64) and the reference row t_i(k')
    double tmax = -CUDART_INF;
    float u2max = 0.f;
    for (int kc = tid; kc < K; kc += NT) {
      float zr[D];
#pragma unroll
      for (int r = 0; r < D; ++r) zr[r] = a.z[((size_t)i * D + r) * K + kc];
      double lq = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const double dz = (double)zr[r] - qconst[r];
        lq += qconst[2 * QEM_MAX_D + r] - dz * dz * qconst[QEM_MAX_D + r];
      }
      double ll;
      if constexpr (OBS == QEM_OBS_GAUSS) {
        const double zz = zr[0];
        ll = ostat[2] - (ostat[1] - 2.0 * zz * ostat[0] + (double)J * zz * zz) * ostat[3];
      } else {
        ll = 0.0;
        for (int j = 0; j < J; ++j) {
          const uint32_t mk = bmask[j];
          float eta = 0.f;
#pragma unroll
          for (int r = 0; r < D; ++r)
            if ((mk >> r) & 1u) eta += zr[r];
          const float sp = fmaxf(eta, 0.f) + log1pf(__expf(-fabsf(eta)));
          ll += (ybits[j] ? (double)eta : 0.0) - (double)sp;
        }
      }
      float U2 = 0.f;
      double U2d = 0.0;
      float* cp = col + (size_t)kc * CS;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const float u = zr[r] - ref.mu_ref[r];
        cp[r] = u;
        U2 = fmaf(u, u, U2);
        U2d += (double)u * (double)u;
      }
      cp[D] = U2;
      const double t = ref.bref_const - 0.5 * ref.e_ref * U2d + (ll - lq);
      tref[kc] = t;
      tmax = fmax(tmax, t);
      u2max = fmaxf(u2max, U2);
    }
    const double M = block_max(tmax, scratch);
    const float U2max = (float)block_max((double)u2max, scratch);
    double s = 0.0;
    for (int kc = tid; kc < K; kc += NT) s += (double)expf((float)(tref[kc] - M));
    const double S = block_sum(s, scratch);
    const double logS = log(S);
    for (int kc = tid; kc < K; kc += NT) {
      const float lp = (float)(tref[kc] - M - logS);
      float* cp = col + (size_t)kc * CS;
      cp[D + 1] = expf(lp);
      cp[D + 2] = lp;
      a.ws.lnP[(size_t)i * K + kc] = lp;
    }
    if (tid == 0) {
      const double ci = M + logS - logK;
      a.ws.cvec[i] = ci;
      csum += ci;
    }
    __syncthreads();

    // ---- pair tile: dg_i(k) for the owned rows, warp-uniform mode
    const float umax = sqrtf(U2max);
    float tb = 0.f;
#pragma unroll
    for (int j = 0; j < 2 * RP; ++j) tb = fmaxf(tb, rb_a[j] + rb_g[j] * U2max + rb_c[j] * umax);
    int md = tb <= 0.0625f ? 0 : (tb <= 0.5f ? 1 : 2);
    md = __reduce_max_sync(0xffffffffu, md);
    float dgv[2 * RP];
    if (md == 0)
      tile_poly<D, RP, 5>(col, Kp, al, ga, cc, dgv);
    else if (md == 1)
      tile_poly<D, RP, 9>(col, Kp, al, ga, cc, dgv);
    else
      tile_online<D, RP>(col, Kp, al, ga, cc, dgv);
#pragma unroll
    for (int j = 0; j < 2 * RP; ++j) {
      if (kid[j] >= 0) {
        a.ws.dg[(size_t)i * K + kid[j]] = dgv[j];
        G[j] += (double)dgv[j];
      }
    }
  }

  // ---- per-CTA partial plate sums, then the last CTA reduces them in order.
  double* part = a.ws.partial + (size_t)blockIdx.x * (K + 1);
#pragma unroll
  for (int j = 0; j < 2 * RP; ++j)
    if (kid[j] >= 0) part[kid[j]] = G[j];
  if (tid == 0) part[K] = csum;
  __threadfence();
  __syncthreads();
  __shared__ uint32_t s_last;
  if (tid == 0) s_last = (atomicAdd(&a.cnt->ticket_fwd, 1u) == gridDim.x - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int k = tid; k <= K; k += NT) {
      double sum = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(a.ws.partial + (size_t)b * (K + 1) + k);
      a.ws.red[k] = sum;
    }
    if (tid == 0) a.cnt->ticket_fwd = 0;
  }
}

