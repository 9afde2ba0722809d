// qem_tl_d24.cu -- the two-level kernels for latent dimension d = 24 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(24)
}  // namespace qem
