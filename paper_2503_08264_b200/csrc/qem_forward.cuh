// qem_forward.cuh -- K2: unary terms + pair-tile forward log-sum-exp for
// two-level models (included inside namespace qem by qem_two_level.cu; needs
// TLArgs, pad4, inv_fact, expm1_poly).
//
// K2a k_colprep  (one warp per group, persistent): for every column k'
//     A_i(k') = sum_j log p(x_ij|z^k') - log q(z^k')            (fp64)
//     t_i(k') = B(k_ref,k') + A_i(k')                            (fp64)
//     c_i = lse_k' t_i - log K;  P_i = softmax t_i;  u = z - mu_ref
//   -> column record colrec[i][k'] = {w[D], |w|^2, P_i, ln P_i} (fp32), w = z - m_i,
//      cvec[i] = c_i, gstat[i] = max |w|^2.
// K2b k_forward  (persistent, TMA double-buffered): the group's column
//   records arrive in shared memory by cp.async.bulk (mbarrier completion)
//   while the previous group's tile is computed; rows k live in registers
//   (sorted by coefficient magnitude so a warp's rows share a mode):
//     dg_i(k) = alpha'_k + log sum_k' P_i(k') exp(D'_k(k')), D' re-centred on the
//     group's Q mean, by
//       modes 0-4: log1p(sum P expm1_n(D')), n = 3/4/5/7/9 while the Taylor
//                  remainder at bound(|D'|), times N groups, stays <= 2e-6
//       mode 5:    single-pass online log-sum-exp of D' + ln P (ex2 on the SFU)
//   The mode is CTA-uniform (max over the CTA's rows) so warps stay in step.
#pragma once

#ifndef QEM_FWD_CH
#define QEM_FWD_CH 16
#endif
template <int D>
struct FwdLayout {
  static constexpr int CS = pad4(D + 3);  // floats per column: u[D], U2, P, lnP
  // field ids after u[0 .. D-1], and each field's float offset in the group's block.  d = 1 lays
  // columns out in pairs, [u0 lnP0 u1 lnP1 | U2_0 P0 U2_1 P1], so the online tile reads both fields
  // of two columns with one 16-byte load.
  static constexpr int FU2 = D, FP = D + 1, FLP = D + 2;
  __host__ __device__ static int off(int kc, int f) {
    if (D == 1) {
      const int slot = f == 0 ? 0 : (f == FLP ? 1 : (f == FU2 ? 2 : 3));
      return (kc >> 1) * 8 + (slot >> 1) * 4 + (kc & 1) * 2 + (slot & 1);
    }
    return kc * CS + f;
  }
  static constexpr int CH = QEM_FWD_CH;   // column chunk of the online log-sum-exp (one max per chunk)
  __host__ __device__ static int kpad(int K) { return (K + CH - 1) / CH * CH; }
  // group trailer after the Kp column records: [0] max |w|^2, [2..3] c_i (fp64), [4..4+D) Q mean m_i
  // (fp32), so the forward's per-group scalars arrive with the group's TMA copy instead of as
  // dependent global loads at the top of every group
  static constexpr int GH = 4 + pad4(D);
  __host__ __device__ static size_t group_floats(int K) { return (size_t)kpad(K) * CS + GH; }
  __host__ __device__ static size_t stage_bytes(int K) { return group_floats(K) * sizeof(float); }
  // k_forward: two stages + two mbarriers + the CTA's plate-sum accumulators (K + 1 Fx2: per row, + c_i)
  // (+ for d = 1 the moment tiles' per-warp partial moments, [warps <= K/64][2 NMAX])
  static constexpr int NMAX = 9;  // highest Taylor degree of the polynomial modes
  __host__ __device__ static size_t mom_bytes(int K) { return D == 1 ? (size_t)((K + 63) / 64) * 2 * NMAX * 8 : 0; }
  __host__ __device__ static size_t bytes(int K, int /*J*/) {
    return 2 * stage_bytes(K) + 16 + (size_t)(K + 1) * 16 + mom_bytes(K);
  }
  // k_colprep, per warp: tref[K] + qconst[3][D] + bern masks/labels [2J]
  __host__ __device__ static size_t prep_warp_bytes(int K, int J) {
    size_t b = (size_t)K * sizeof(double) + 3 * D * sizeof(double) + (size_t)2 * J * sizeof(uint32_t);
    return (b + 15) & ~(size_t)15;
  }
  static constexpr int PREP_WARPS = 8;
  __host__ __device__ static size_t prep_bytes(int K, int J) { return PREP_WARPS * prep_warp_bytes(K, J); }
};

// D'_k(k') + base: the column term `base` (0, or ln P in the online tile) rides in the contraction's
// first FMA instead of a separate add
template <int D, int RP>
__device__ __forceinline__ float2 pair_D(float2 base, const float2 (&ga)[RP], const float2 (&cc)[RP][D],
                                         int p, const float* u, float U2) {
  if constexpr (D == 1) {
    return fma2(fma2(ga[p], f2(u[0]), cc[p][0]), f2(u[0]), base);
  } else {
    // two accumulators halve the dependent FMA chain
    float2 a0 = fma2(ga[p], f2(U2), base);
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

// column kc's fields (col = the group's block)
template <int D>
__device__ __forceinline__ void load_col(const float* col, int kc, float (&u)[D], float& U2, float& P, float& lnP) {
  if constexpr (D == 1) {
    u[0] = col[FwdLayout<1>::off(kc, 0)];
    U2 = col[FwdLayout<1>::off(kc, FwdLayout<1>::FU2)];
    P = col[FwdLayout<1>::off(kc, FwdLayout<1>::FP)];
    lnP = col[FwdLayout<1>::off(kc, FwdLayout<1>::FLP)];
    return;
  }
  constexpr int CS = pad4(D + 3);
  const float* cr = col + (size_t)kc * CS;
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
  U2 = buf[FwdLayout<D>::FU2];
  P = buf[FwdLayout<D>::FP];
  lnP = buf[FwdLayout<D>::FLP];
}

__device__ __forceinline__ float2 max2(float2 a, float2 b) { return make_float2(fmaxf(a.x, b.x), fmaxf(a.y, b.y)); }

template <int D, int RP, int N>
__device__ __forceinline__ void tile_poly(const float* col, int Kp, const float2 (&ga)[RP],
                                          const float2 (&cc)[RP][D], double (&dgv)[2 * RP]) {
  constexpr int CS = pad4(D + 3);
  float2 acc[RP];
#pragma unroll
  for (int p = 0; p < RP; ++p) acc[p] = f2(0.f);
#pragma unroll 2
  for (int kc = 0; kc < Kp; ++kc) {
    float u[D], U2, P, lnP;
    load_col<D>(col, kc, u, U2, P, lnP);
#pragma unroll
    for (int p = 0; p < RP; ++p) acc[p] = fma2(f2(P), expm1_poly<N>(pair_D<D, RP>(f2(0.f), ga, cc, p, u, U2)), acc[p]);
  }
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    dgv[2 * p] = log1p((double)acc[p].x);  // fp64 logs: the fp32 ones' ~1-ulp errors are not zero-mean,
    dgv[2 * p + 1] = log1p((double)acc[p].y);  // and they add up coherently over the groups' plate sum
  }
}

// Polynomial modes for d = 1 through the group's column moments.  With D'_k(k') = g_k w^2 + c_k w
// (w = w(k'), the row's re-centred coefficients), the degree-N Taylor sum of tile_poly is
//   sum_k' P(k') expm1_N(D'_k(k')) = sum_{n=1..N} (1/n!) sum_{j=0..n} C(n,j) g_k^j c_k^(n-j) mu_{n+j},
//   mu_p = sum_k' P(k') w(k')^p   (p = 1 .. 2N, the same for every row of the group),
// the same polynomial rearranged (exact algebra): O(K N) moments + O(N^2) per row instead of O(N) per
// pair, all in fp64.  No cancellation beyond the Taylor terms' own size: the mode's bound tb >=
// |c_k| max|w| + |g_k| max w^2 bounds every expanded term by tb^n.  The moments are reduced in a
// fixed order (warp butterflies, then warps in index order), so the result is deterministic.
template <int N>
__device__ __forceinline__ double poly_from_moments(double g, double c, const double* mu) {
  double gp[N + 1], cp[N + 1];
  gp[0] = 1.0;
  cp[0] = 1.0;
#pragma unroll
  for (int j = 1; j <= N; ++j) {
    gp[j] = gp[j - 1] * g;
    cp[j] = cp[j - 1] * c;
  }
  double acc = 0.0, fact = 1.0;
#pragma unroll
  for (int n = 1; n <= N; ++n) {
    fact *= n;
    double sn = 0.0, bin = 1.0;  // C(n, j)
#pragma unroll
    for (int j = 0; j <= n; ++j) {
      sn = fma(bin * gp[j] * cp[n - j], mu[n + j - 1], sn);
      bin = bin * (n - j) / (j + 1);
    }
    acc = fma(sn, 1.0 / fact, acc);
  }
  return acc;
}

template <int RP, int N>
__device__ __forceinline__ void tile_moments1(const float* col, int K, const float2 (&ga)[RP], const float2 (&cc)[RP][1],
                                              double (&dgv)[2 * RP], double* s_mom) {
  constexpr int CS = pad4(4), NM = 2 * N;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  double m[NM];
#pragma unroll
  for (int p = 0; p < NM; ++p) m[p] = 0.0;
  for (int kc = tid; kc < K; kc += blockDim.x) {
    const double w = col[FwdLayout<1>::off(kc, 0)], P = col[FwdLayout<1>::off(kc, FwdLayout<1>::FP)];
    double pw = P;
#pragma unroll
    for (int p = 0; p < NM; ++p) {
      pw *= w;
      m[p] += pw;
    }
  }
#pragma unroll
  for (int p = 0; p < NM; ++p) m[p] = warp_sum(m[p]);
  if (lane == 0)
#pragma unroll
    for (int p = 0; p < NM; ++p) s_mom[wid * NM + p] = m[p];
  __syncthreads();
  double mu[NM];
#pragma unroll
  for (int p = 0; p < NM; ++p) mu[p] = 0.0;
  for (int w = 0; w < nw; ++w)
#pragma unroll
    for (int p = 0; p < NM; ++p) mu[p] += s_mom[w * NM + p];
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    dgv[2 * p] = log1p(poly_from_moments<N>((double)ga[p].x, (double)cc[p][0].x, mu));
    dgv[2 * p + 1] = log1p(poly_from_moments<N>((double)ga[p].y, (double)cc[p][0].y, mu));
  }
}

// 1 = d = 1 polynomial modes through the column moments (tile_moments1), 0 = per pair (tile_poly)
#ifndef QEM_MOMENT_TILES
#define QEM_MOMENT_TILES 1
#endif
constexpr bool kMomentTiles = QEM_MOMENT_TILES != 0;

template <int D, int RP, int N>
__device__ __forceinline__ void tile_poly_mode(const float* col, int K, int Kp, const float2 (&ga)[RP],
                                               const float2 (&cc)[RP][D], double (&dgv)[2 * RP], double* s_mom) {
  if constexpr (D == 1 && kMomentTiles)
    tile_moments1<RP, N>(col, K, ga, cc, dgv, s_mom);
  else
    tile_poly<D, RP, N>(col, Kp, ga, cc, dgv);
}

// Exponentials per online chunk (the last fwd_soft<D>() of its QEM_FWD_CH columns) evaluated on the FMA
// pipe (exp2_poly2) instead of the SFU.  Narrow latents (d <= 4: the contraction leaves the FMA pipe
// half idle next to the SFU) take 2 of 16 (config 4, interleaved A/B: 0 1.886, 2 1.796, 3 1.816,
// 4 1.847, 6 2.052 ms per forward); wide ones none.  QEM_FWD_SOFT overrides.
template <int D>
__host__ __device__ constexpr int fwd_soft() {
#ifdef QEM_FWD_SOFT
  return QEM_FWD_SOFT;
#else
  return D <= 4 ? 2 : 0;
#endif
}

// Rescale margin of the online log-sum-exp (natural-log units).  0 = the shift is always the exact
// running max, so the dominant term of every row is ex2(0) = 1 exactly: a positive margin saves
// rescales but leaves ~1e-7 relative error on the dominant term, which the 1e5-group plate sum of
// config 4 random-walks past the weight tolerance (tests/test_gpu_fullsize.py, intermediate regime).
constexpr float kLazy = 0.0f;

template <int D, int RP>
__device__ __forceinline__ void tile_online(const float* col, int Kp, const float2 (&ga)[RP],
                                            const float2 (&cc)[RP][D], double (&dgv)[2 * RP]) {
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
    if constexpr (D == 1) {  // two columns' (w, ln P) per 16-byte load; ln P rides in the last FMA
#pragma unroll
      for (int c = 0; c < CH; c += 2) {
        const float4 v = *reinterpret_cast<const float4*>(col + (size_t)((kc0 + c) >> 1) * 8);
        const float u0[1] = {v.x}, u1[1] = {v.z};
#pragma unroll
        for (int p = 0; p < RP; ++p) {
          tv[c][p] = pair_D<D, RP>(f2(v.y), ga, cc, p, u0, 0.f);
          tv[c + 1][p] = pair_D<D, RP>(f2(v.w), ga, cc, p, u1, 0.f);
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float u[D], U2, P, lnP;
        load_col<D>(col, kc0 + c, u, U2, P, lnP);
#pragma unroll
        for (int p = 0; p < RP; ++p) tv[c][p] = add2(pair_D<D, RP>(f2(0.f), ga, cc, p, u, U2), f2(lnP));
      }
    }
#pragma unroll
    for (int p = 0; p < RP; ++p) {
      float2 cm = tv[0][p];
#pragma unroll
      for (int c = 1; c < CH; ++c) cm = max2(cm, tv[c][p]);
      // rescale only when a chunk raises the running max (rare after the first chunks)
      if (cm.x > mr[p].x + kLazy) {
        ac[p].x *= ex2((mr[p].x - cm.x) * kLog2e);
        mr[p].x = cm.x;
      }
      if (cm.y > mr[p].y + kLazy) {
        ac[p].y *= ex2((mr[p].y - cm.y) * kLog2e);
        mr[p].y = cm.y;
      }
      const float2 nm = make_float2(-mr[p].x * kLog2e, -mr[p].y * kLog2e);
      float2 s = ac[p];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const float2 e = fma2(tv[c][p], f2(kLog2e), nm);
        s = add2(s, c >= CH - fwd_soft<D>() ? exp2_poly2(e) : make_float2(ex2(e.x), ex2(e.y)));
      }
      ac[p] = s;
    }
  }
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    // the row's dominant term is ex2(0) = 1, so ac >= 1 (finite unless the inputs were not)
    dgv[2 * p] = (double)mr[p].x + (isfinite(ac[p].x) ? log_pos_f32(ac[p].x) : log((double)ac[p].x));
    dgv[2 * p + 1] = (double)mr[p].y + (isfinite(ac[p].y) ? log_pos_f32(ac[p].y) : log((double)ac[p].y));
  }
}

// ------------------------------------------------------------------ K2a
// One WARP per group (warp-shuffle reductions only, no block barriers); the
// CTA's warps work on different groups.
template <int D, int OBS, bool TC_UNUSED>
__global__ void __launch_bounds__(256) k_colprep(TLArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int CS = pad4(D + 3);
  const int K = a.K, J = a.J, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int Kp = FwdLayout<D>::kpad(K);
  unsigned char* wbase = smem + (size_t)wid * FwdLayout<D>::prep_warp_bytes(K, J);
  double* tref = reinterpret_cast<double*>(wbase);      // [K]
  double* qconst = tref + K;                            // [3][D]
  uint32_t* bmask = reinterpret_cast<uint32_t*>(qconst + 3 * D);  // [J]
  uint32_t* ybits = bmask + J;                          // [J]
  // reference-row constants (fields read individually: the struct is large)
  float mu_ref[D];
#pragma unroll
  for (int r = 0; r < D; ++r) mu_ref[r] = a.ws.ref->mu_ref[r];
  const double bref_const = a.ws.ref->bref_const, e_ref = a.ws.ref->e_ref;
  const double logK = log((double)K);
  double gc0 = 0.0, gc1 = 0.0;
  if constexpr (OBS == QEM_OBS_GAUSS) {
    gc0 = -0.5 * J * (kLn2Pi + log(a.obs_var));
    gc1 = 0.5 / a.obs_var;
  }
  for (int64_t i = (int64_t)blockIdx.x * nwarps + wid; i < a.n_local; i += (int64_t)gridDim.x * nwarps) {
    __syncwarp();
    if (lane < D) {
      const double m = a.q_m[i * D + lane], v = a.q_v[i * D + lane];
      qconst[lane] = m;
      qconst[D + lane] = 0.5 / v;
      qconst[2 * D + lane] = -0.5 * (kLn2Pi + log(v));
    }
    double sx = 0.0, sxx = 0.0;
    if constexpr (OBS == QEM_OBS_GAUSS) {
      const float* x = reinterpret_cast<const float*>(a.x) + i * J;
      for (int j = lane; j < J; j += 32) {
        const double xv = x[j];
        sx += xv;
        sxx += xv * xv;
      }
      sx = warp_sum(sx);
      sxx = warp_sum(sxx);
    } else {
      const uint8_t* x = reinterpret_cast<const uint8_t*>(a.x) + (size_t)i * J * D;
      const uint8_t* y = reinterpret_cast<const uint8_t*>(a.y) + (size_t)i * J;
      for (int j = lane; j < J; j += 32) {
        uint32_t mk = 0;
#pragma unroll
        for (int r = 0; r < D; ++r) mk |= (x[j * D + r] ? 1u : 0u) << r;
        bmask[j] = mk;
        ybits[j] = y[j] ? 1u : 0u;
      }
    }
    __syncwarp();
    float* rec0 = a.ws.colrec + (size_t)i * FwdLayout<D>::group_floats(K);
    double tmax = -CUDART_INF;
    float u2max = 0.f;
    for (int kc = lane; kc < K; kc += 32) {
      float zr[D];
#pragma unroll
      for (int r = 0; r < D; ++r) zr[r] = a.z[((size_t)i * D + r) * K + kc];
      double lq = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const double dz = (double)zr[r] - qconst[r];
        lq += qconst[2 * D + r] - dz * dz * qconst[D + r];
      }
      double ll;
      if constexpr (OBS == QEM_OBS_GAUSS) {
        const double zz = zr[0];
        ll = gc0 - (sxx - 2.0 * zz * sx + (double)J * zz * zz) * gc1;
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
      // record the group-centred offsets w = z - m_i (DESIGN.md "Forward":
      // recentring); the reference row uses u = z - mu_ref exactly in fp64.
      float rec[CS];
      float W2 = 0.f;
      double U2d = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const float w = zr[r] - (float)qconst[r];
        rec[r] = w;
        W2 = fmaf(w, w, W2);
        const double u = (double)zr[r] - (double)mu_ref[r];
        U2d += u * u;
      }
      if constexpr (D == 1) {  // pair layout: (w, ln P) and (U2, P) are 8-byte halves (P, ln P below)
        *reinterpret_cast<float2*>(rec0 + FwdLayout<1>::off(kc, 0)) = make_float2(rec[0], 0.f);
        *reinterpret_cast<float2*>(rec0 + FwdLayout<1>::off(kc, FwdLayout<1>::FU2)) = make_float2(W2, 0.f);
      } else {
#pragma unroll
        for (int r = D; r < CS; ++r) rec[r] = 0.f;
        rec[FwdLayout<D>::FU2] = W2;
        float4* dst = reinterpret_cast<float4*>(rec0 + (size_t)kc * CS);
#pragma unroll
        for (int q = 0; q < CS / 4; ++q)
          dst[q] = make_float4(rec[4 * q], rec[4 * q + 1], rec[4 * q + 2], rec[4 * q + 3]);
      }
      const double t = bref_const - 0.5 * e_ref * U2d + (ll - lq);
      a.ws.tA[(size_t)i * K + kc] = t;  // t_ref, for the backward's k*-row softmax
      tref[kc] = t;
      tmax = fmax(tmax, t);
      u2max = fmaxf(u2max, W2);
    }
    // padding columns: P = 0, ln P = -inf (contribute nothing)
    {
      for (int kc = K + lane; kc < Kp; kc += 32) {
#pragma unroll
        for (int f = 0; f < D + 3; ++f) rec0[FwdLayout<D>::off(kc, f)] = 0.f;
        rec0[FwdLayout<D>::off(kc, FwdLayout<D>::FLP)] = -CUDART_INF_F;
      }
    }
    const double M = warp_max(tmax);
    const float U2max = warp_maxf(u2max);
    double s = 0.0;
    for (int kc = lane; kc < K; kc += 32) s += (double)expf((float)(tref[kc] - M));
    const double logS = log(warp_sum(s));
    for (int kc = lane; kc < K; kc += 32) {
      const float lp = (float)(tref[kc] - M - logS);
      {
        rec0[FwdLayout<D>::off(kc, FwdLayout<D>::FP)] = expf(lp);
        rec0[FwdLayout<D>::off(kc, FwdLayout<D>::FLP)] = lp;
      }
    }
    if (lane == 0) {
      const double cv = M + logS - logK;
      a.ws.cvec[i] = cv;
      a.ws.gstat[i] = U2max;
      float* gh = rec0 + (size_t)Kp * CS;
      gh[0] = U2max;
      gh[1] = 0.f;
      *reinterpret_cast<double*>(gh + 2) = cv;
    }
    if (lane < D) rec0[(size_t)Kp * CS + 4 + lane] = a.q_m[i * D + lane];
  }
}

// ------------------------------------------------------------------ K2b
// Thread t owns the row slots s = 2(t*RP+p)+h (p < RP float2 pairs), i.e.
// rows k = perm[s].  Per group the row coefficients are re-centred on the
// group's Q mean m_i (u = u0 + w, u0 = m_i - mu_ref, w = z - m_i):
//   D_k(k') = alpha'_k + gamma_k |w|^2 + c'_k . w,
//   alpha'_k = alpha_k + gamma_k |u0|^2 + c_k . u0,   c'_k = c_k + 2 gamma_k u0,
// so the column loop only sees the small within-group part and alpha'_k is
// added back to dg at the end (exact algebra).
template <int D, int RP>
// Register budget (min resident blocks of 256 threads): d <= 4 runs 2 rows per thread in <= 64
// registers (config 4: 8 CTAs of 128 threads = 32 warps per SM; 4 rows in 124 registers at 8 CTAs of 64 measured
// 1.998 ms against 1.886), wider latents keep the 128-register budget.  QEM_FWD_MINB overrides.
#ifdef QEM_FWD_MINB
__global__ void __launch_bounds__(256, QEM_FWD_MINB) k_forward(TLArgs a) {
#else
__global__ void __launch_bounds__(256, (D <= 4 && RP == 1) ? 4 : 2) k_forward(TLArgs a) {
#endif
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int CS = pad4(D + 3);
  constexpr int CW = D + 2;
  const int K = a.K, tid = threadIdx.x;
  const int Kp = FwdLayout<D>::kpad(K);
  const uint32_t sbytes = (uint32_t)FwdLayout<D>::stage_bytes(K);
  // stage s lives at smem + s*sbytes (pointer arithmetic on the __shared__ symbol keeps LDS addressing)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * sbytes);

  float mur[D];
#pragma unroll
  for (int r = 0; r < D; ++r) mur[r] = a.ws.ref->mu_ref[r];
  int kid[2 * RP];
  float2 ga[RP];
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    float gv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * (tid * RP + p) + h;  // a warp owns a contiguous run of sorted slots
      const bool ok = s < K;
      const int k = ok ? a.ws.perm[s] : 0;
      kid[2 * p + h] = ok ? k : -1;
      gv[h] = ok ? a.ws.fwd_coef[(size_t)k * CW + 1] : 0.f;
    }
    ga[p] = make_float2(gv[0], gv[1]);
  }
  // plate-sum accumulators in shared memory (a thread owns its rows' entries; registers are the
  // tile's): G[k] for row k, G[K] for sum_i c_i
  Fx2* G = reinterpret_cast<Fx2*>(smem + 2 * sbytes + 16);
  double* s_mom = reinterpret_cast<double*>(smem + 2 * sbytes + 16 + (size_t)(K + 1) * 16);  // d = 1 moment tiles
#pragma unroll
  for (int q = 0; q < 2 * RP; ++q)
    if (kid[q] >= 0) G[kid[q]] = Fx2{};
  if (tid == 0) G[K] = Fx2{};
  uint32_t mc0 = 0, mc1 = 0, mc2 = 0, mc3 = 0, mc4 = 0, mc5 = 0;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t i0 = blockIdx.x;
  if (tid == 0 && i0 < a.n_local) {
    mbar_expect_tx(&bar[0], sbytes);
    tma_bulk_g2s(smem, a.ws.colrec + (size_t)i0 * FwdLayout<D>::group_floats(K), sbytes, &bar[0]);
  }
  __shared__ int s_mode[2][8];
  __shared__ float s_tb[2][8];  // d = 1: per-warp |D'| bounds (the backward's moment-tile decision)
  // Groups past the first wave come from a device-wide queue (one atomic per group): per-group cost
  // depends on the tile mode, so a static stride leaves CTAs idle at the end of the launch.
  __shared__ int64_t s_next[2];
  int j = 0;
  for (int64_t i = i0; i < a.n_local; ++j) {
    const int st = j & 1;
    if (tid == 0) s_next[st] = (int64_t)gridDim.x + atomicAdd(&a.cnt->claim_fwd, 1u);
    // the group's records (issued one group ago) carry its scalars in the trailer
    mbar_wait(&bar[st], (uint32_t)((j >> 1) & 1));
    const float* col = reinterpret_cast<const float*>(smem + (st ? sbytes : 0));
    const float* gh = col + (size_t)Kp * CS;
    const float W2max = gh[0];
    if (tid == 0) G[K].add(*reinterpret_cast<const double*>(gh + 2));

    // ---- re-centred row coefficients for this group (before the barrier, so
    // the CTA-wide tile mode costs no extra synchronisation)
    float u0[D];
    float U0sq = 0.f;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      u0[r] = gh[4 + r] - mur[r];
      U0sq = fmaf(u0[r], u0[r], U0sq);
    }
    const float wmax = sqrtf(W2max);
    // alpha'_k in fp64 (it can be large where D is large; the tile only sees D')
    double ald[2 * RP];
    float2 cc[RP][D];
    float tb = 0.f;
#pragma unroll
    for (int p = 0; p < RP; ++p) {
      float cv[2][D];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = kid[2 * p + h] >= 0 ? kid[2 * p + h] : 0;
        const float* fc = a.ws.fwd_coef + (size_t)k * CW;
        const float g = h ? ga[p].y : ga[p].x;
        double ap = a.ws.alpha_d[k] + (double)g * (double)U0sq;
        float cn = 0.f;
#pragma unroll
        for (int r = 0; r < D; ++r) {
          const float c = fc[2 + r];
          ap += (double)c * (double)u0[r];
          cv[h][r] = fmaf(2.f * g, u0[r], c);
          cn = fmaf(cv[h][r], cv[h][r], cn);
        }
        ald[2 * p + h] = ap;
        tb = fmaxf(tb, sqrtf(cn) * wmax + fabsf(g) * W2max);
      }
#pragma unroll
      for (int r = 0; r < D; ++r) cc[p][r] = make_float2(cv[0][r], cv[1][r]);
    }
    // degree n of the expm1 Taylor polynomial such that its remainder at the
    // bound, summed over all N groups, stays below 2e-6
    int md = tb <= a.thr[0] ? 0 : (tb <= a.thr[1] ? 1 : (tb <= a.thr[2] ? 2 : (tb <= a.thr[3] ? 3 : (tb <= a.thr[4] ? 4 : 5))));
    md = __reduce_max_sync(0xffffffffu, md);
    if ((tid & 31) == 0) s_mode[st][tid >> 5] = md;
    if constexpr (D == 1) {  // tb >= 0: its bits order like unsigned integers
      const float tbw = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(tb)));
      if ((tid & 31) == 0) s_tb[st][tid >> 5] = tbw;
    }

    // all warps are done with the other stage (group j-1): refill it with group j+1
    __syncthreads();
    const int64_t inext = s_next[st];
    if (tid == 0 && inext < a.n_local) {
      mbar_expect_tx(&bar[st ^ 1], sbytes);
      tma_bulk_g2s(smem + (st ? 0 : sbytes), a.ws.colrec + (size_t)inext * FwdLayout<D>::group_floats(K), sbytes,
                   &bar[st ^ 1]);
    }
    // CTA-uniform mode: every warp does the same work per group (no barrier skew)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) md = max(md, s_mode[st][w]);
    if constexpr (D == 1) {
      if (tid == 0) {
        float tbg = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tbg = fmaxf(tbg, s_tb[st][w]);
        a.ws.gtb[i] = tbg;
      }
    }
    mc0 += md == 0;
    mc1 += md == 1;
    mc2 += md == 2;
    mc3 += md == 3;
    mc4 += md == 4;
    mc5 += md == 5;
    double dgv[2 * RP];
    switch (md) {
      case 0: tile_poly_mode<D, RP, 3>(col, K, Kp, ga, cc, dgv, s_mom); break;
      case 1: tile_poly_mode<D, RP, 4>(col, K, Kp, ga, cc, dgv, s_mom); break;
      case 2: tile_poly_mode<D, RP, 5>(col, K, Kp, ga, cc, dgv, s_mom); break;
      case 3: tile_poly_mode<D, RP, 7>(col, K, Kp, ga, cc, dgv, s_mom); break;
      case 4: tile_poly_mode<D, RP, 9>(col, K, Kp, ga, cc, dgv, s_mom); break;
      default: tile_online<D, RP>(col, Kp, ga, cc, dgv); break;
    }
    // h = log sum P exp(D') feeds the backward directly (no cancellation against
    // alpha'); dg = alpha' + h in fp64 feeds the plate sum.
#pragma unroll
    for (int q = 0; q < 2 * RP; ++q) {
      if (kid[q] >= 0) {
        const double dgd = ald[q] + dgv[q];
        a.ws.hmsg[(size_t)i * K + kid[q]] = (float)dgv[q];
        a.ws.dg[(size_t)i * K + kid[q]] = (float)dgd;
        G[kid[q]].add(dgd);
      }
    }
    i = inext;
  }

  // ---- plate sums: each CTA adds its rows' split sums (Fx2) into the (K + 1) x {h, m} accumulators
  // k_root_prep zeroed; the parts are exact sums on fixed grids, so the atomics' order (which CTA
  // drew which groups from the queue, which CTA adds first) cannot change a bit (R39), and
  // no CTA has to walk every CTA's partials at the end (1184 of them on config 4).
  double* acc_h = a.ws.partial;
  double* acc_m = a.ws.partial + (K + 1);
#pragma unroll
  for (int q = 0; q < 2 * RP; ++q)
    if (kid[q] >= 0) {
      atomicAdd(&acc_h[kid[q]], G[kid[q]].h);
      atomicAdd(&acc_m[kid[q]], G[kid[q]].m);
    }
  if (tid == 0) {
    atomicAdd(&acc_h[K], G[K].h);
    atomicAdd(&acc_m[K], G[K].m);
  }
  if ((tid & 31) == 0)
  {
    const uint32_t mcs[6] = {mc0, mc1, mc2, mc3, mc4, mc5};
#pragma unroll
    for (int m = 0; m < 6; ++m)
      if (mcs[m]) atomicAdd(&a.cnt->mode_hist[m], (unsigned long long)mcs[m]);
  }
  __threadfence();
  __syncthreads();
  __shared__ uint32_t s_last;
  if (tid == 0) s_last = (atomicAdd(&a.cnt->ticket_fwd, 1u) == gridDim.x - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int k = tid; k <= K; k += blockDim.x) a.ws.red[k] = __ldcg(acc_h + k) + __ldcg(acc_m + k);
    if (tid == 0) {
      a.cnt->ticket_fwd = 0;
      a.cnt->claim_fwd = 0;
    }
  }
}
