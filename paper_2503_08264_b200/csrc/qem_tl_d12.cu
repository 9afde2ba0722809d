// qem_tl_d12.cu -- the two-level kernels for latent dimension d = 12 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(12)
}  // namespace qem
