// qem_two_level.cu -- dispatch of the two-level MPIW E-step on the runtime latent dimension d
// (configs 1, 2, 4, 5).  The kernels are templated on D (qem_two_level.cuh); every D of the menu
// below is compiled in its own translation unit qem_tl_d<D>.cu.  A model whose d is not on the menu
// is rejected by qem_model_validate (QEM_INVALID_MODEL) -- the menu is QEM_D_MENU in include/qem.h.
#include <cstdlib>

#include "qem_internal.h"

namespace qem {

#define QEM_D_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10) X(12) X(14) X(16) X(18) X(20) X(24) X(32)

// per-D entry points, explicitly instantiated in qem_tl_d<D>.cu
template <int D>
cudaError_t tl_forward_d(qem_ctx*, cudaStream_t);
template <int D>
cudaError_t tl_backward_d(qem_ctx*, cudaStream_t);
template <int D>
void tl_grids_d(const qem_model_desc*, int64_t, int, int*, int*, int*);
template <int D>
size_t tl_max_smem_d(const qem_model_desc*);

constexpr int kTcD = 16;  // the tensor-core contraction width (qem_tc.cuh)

int tl_supported_d(int d) {
#define X(v) if (d == v) return 1;
  QEM_D_LIST(X)
#undef X
  return 0;
}

int tl_use_tc(const qem_model_desc* d) {
  static const int off = getenv("QEM_NO_TC") != nullptr;  // tuning / comparison override
  // tensor-core pair kernels, K a multiple of 256: 8 <= d <= 16 with Bernoulli-logit observations
  // (split layout, contraction zero-padded to 16), or d = 1 with Gaussian ones (compact layout).
  // For 2 <= d < 8 the FFMA tiles stay: the split layout's 128-byte column operand would be mostly
  // padding.
  // d = 1 with Gaussian observations (config 4): the compact layout, one c-region MMA + the extra slab
  // per tile and a 64-byte column operand (compact path) -- opt-in
  // (QEM_TC1=1): on config 4 its forward is faster than the FFMA tiles but the step is not, and the
  // online mode's ln P inside the MMA is biased by the truncating accumulation
  static const int on1 = getenv("QEM_TC1") != nullptr && atoi(getenv("QEM_TC1")) != 0;
  if (off || d->K % 256 != 0 || d->K > QEM_MAX_K) return 0;
  if (d->d == 1) return on1 && d->obs_kind == QEM_OBS_GAUSS;
  return d->d >= 8 && d->d <= kTcD && tl_supported_d(d->d) && d->obs_kind == QEM_OBS_BERNOULLI_LOGIT;
}

size_t tl_max_smem(const qem_model_desc* d) {
  switch (d->d) {
#define X(v) \
  case v:    \
    return tl_max_smem_d<v>(d);
    QEM_D_LIST(X)
#undef X
  }
  return 0;
}

void tl_grids(const qem_model_desc* d, int64_t n_local, int sms, int* gf, int* gb, int* gp) {
  *gf = *gb = *gp = 1;
  switch (d->d) {
#define X(v)                                   \
  case v:                                      \
    tl_grids_d<v>(d, n_local, sms, gf, gb, gp); \
    return;
    QEM_D_LIST(X)
#undef X
  }
}

cudaError_t tl_forward(qem_ctx* c, cudaStream_t st) {
  switch (c->desc.d) {
#define X(v) \
  case v:    \
    return tl_forward_d<v>(c, st);
    QEM_D_LIST(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

cudaError_t tl_backward(qem_ctx* c, cudaStream_t st) {
  switch (c->desc.d) {
#define X(v) \
  case v:    \
    return tl_backward_d<v>(c, st);
    QEM_D_LIST(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

}  // namespace qem
