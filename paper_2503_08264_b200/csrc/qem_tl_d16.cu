// qem_tl_d16.cu -- the two-level kernels for latent dimension d = 16 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(16)
}  // namespace qem
