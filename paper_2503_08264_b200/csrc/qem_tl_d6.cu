// qem_tl_d6.cu -- the two-level kernels for latent dimension d = 6 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(6)
}  // namespace qem
